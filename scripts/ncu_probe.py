"""A few cfg4 executes for ncu: MODE=full (default) or MODE=pairs (node rows +
class pairs only, no outputs)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_04285_b200 import engine as E, graph as G, models as M

g, t = M.cfg4()
plan = E.Plan(G.flatten(g), t, device=0)
ne, nn = plan.sizes["num_aux_edges"], plan.sizes["num_aux_nodes"]
dev = torch.device("cuda", 0)
outs = {k: torch.empty(ne, dtype=torch.float64, device=dev) for k in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes")}
outs.update({k: torch.empty(nn, dtype=torch.float64, device=dev) for k in ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes")})
mode = os.environ.get("MODE", "full")
cs = E.device_cost_struct(outs) if mode == "full" else E.device_cost_struct({})
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
for i in range(6):
    flush.zero_()
    plan.execute(cs, edge_range=(0, -1) if mode == "full" else (0, 0))
torch.cuda.synchronize()
plan.check_errors()
print("ok", mode)
