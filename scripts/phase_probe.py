"""Time the phases of one cfg4 build through the split API (device-resident):
pairs+nodes only (no edge outputs), full build, and each pair form."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_04285_b200 import engine as E, graph as G, models as M

g, t = M.cfg4()
f = G.flatten(g)
plan = E.Plan(f, t, device=0)
ne, nn = plan.sizes["num_aux_edges"], plan.sizes["num_aux_nodes"]
dev = torch.device("cuda", 0)
outs = {k: torch.empty(ne, dtype=torch.float64, device=dev) for k in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes")}
outs.update({k: torch.empty(nn, dtype=torch.float64, device=dev) for k in ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes")})
full = E.device_cost_struct(outs)
nodes_only = E.device_cost_struct({k: v for k, v in outs.items() if k.startswith("node")})
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
s = torch.cuda.Stream()
plan.upload(s.cuda_stream)

def timeit(cs, n=20, **kw):
    ts = []
    with torch.cuda.stream(s):
        for i in range(n + 3):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            plan.execute(cs, stream=s.cuda_stream, **kw)
            b.record(s)
            if i >= 3:
                ts.append((a, b))
    torch.cuda.synchronize()
    plan.check_errors()
    v = sorted(x.elapsed_time(y) * 1e3 for x, y in ts)
    return v[len(v) // 2]

for form in (1, 2):
    plan.set_pair_form(form)
    print(f"form {form}: nodes+pairs only {timeit(nodes_only):.1f} us, full build {timeit(full):.1f} us, "
          f"nodes only {timeit(full, edge_range=(0, 0)):.1f} us, pairs only {timeit(nodes_only, skip_nodes=True):.1f} us, "
          f"empty {timeit(nodes_only, edge_range=(0, 0), skip_nodes=True):.1f} us")
