"""Fixed cost of one build: event-timed execute of tiny and large graphs, and
an empty kernel launch for reference."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_04285_b200 import engine as E, graph as G, models as M

dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)

def timed(fn, n=30):
    ts = []
    with torch.cuda.stream(s):
        for i in range(n + 3):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
            if i >= 3:
                ts.append((a, b))
    torch.cuda.synchronize()
    v = sorted(x.elapsed_time(y) * 1e3 for x, y in ts)
    return v[len(v) // 2]

x = torch.empty(1, device=dev)
print(f"tiny torch kernel: {timed(lambda: x.add_(1)):.1f} us")
for name in ("cfg1", "cfg2", "cfg4"):
    g, t = getattr(M, name)()
    plan = E.Plan(G.flatten(g), t, device=0)
    sz = plan.sizes
    outs = {k: torch.empty(max(1, sz["num_aux_edges"]), dtype=torch.float64, device=dev)
            for k in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes")}
    outs.update({k: torch.empty(max(1, sz["num_aux_nodes"]), dtype=torch.float64, device=dev)
                 for k in ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes")})
    cs = E.device_cost_struct(outs)
    plan.upload(s.cuda_stream)
    full = timed(lambda: plan.execute(cs, stream=s.cuda_stream))
    plan.set_timeline(True)
    with torch.cuda.stream(s):
        flush.zero_()
        plan.execute(cs, stream=s.cuda_stream)
    tl = plan.timeline()
    plan.set_timeline(False)
    print(f"{name}: aux edges {sz['num_aux_edges']}, entries {sz['num_pair_evals']}, build {full:.1f} us, in-kernel end {tl['end']/1e3:.1f} us")
