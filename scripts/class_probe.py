"""cfg4: per edge class, when its class-table entries finish (device timeline)
and how many aux edges the class owns -- what a class-major fan-out could
overlap with the pricing."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
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
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
s = torch.cuda.Stream()
plan.upload(s.cuda_stream)
plan.set_timeline(True)
with torch.cuda.stream(s):
    for i in range(6):
        flush.zero_()
        plan.execute(full, stream=s.cuda_stream)
torch.cuda.synchronize()
pr, it, fo, prof, wx = plan.timeline_detail()
end = (pr[:, 0] + pr[:, 1]) / 1e3
ix = plan.index()
# aux edges per class: the class of every graph edge from the engine's FanSeg is not exported;
# recompute it from the pairs' class ids through a second pass on edge order
for c in np.unique(pr[:, 2]):
    m = pr[:, 2] == c
    e = end[m]
    cl = prof[m]
    print(f"class {c}: {m.sum()} entries, end p50 {np.percentile(e,50):.1f} p90 {np.percentile(e,90):.1f} max {e.max():.1f} us;"
          f" ops med {np.median(cl[:,3]):.0f} max {cl[:,3].max()}, clocks med {np.median(cl[:,0]+cl[:,1]+cl[:,2]):.0f} max {(cl[:,0]+cl[:,1]+cl[:,2]).max()}"
          f" (closure / axes / inference med {np.median(cl[:,0]):.0f} / {np.median(cl[:,1]):.0f} / {np.median(cl[:,2]):.0f};"
          f" U med {np.median(cl[:,4]):.0f}, depth med {np.median(cl[:,5]):.0f}, rounds med {np.median(cl[:,6]):.0f})")
print("rows end max", ((it[:, 0] + it[:, 1]) / 1e3).max())
print("fan ranges: n", len(fo), "ready p50/max", np.percentile((fo[:,0]+fo[:,1])/1e3, 50), ((fo[:,0]+fo[:,1])/1e3).max(),
      "end max", ((fo[:,0]+fo[:,2])/1e3).max())
# the slowest entries: start, duration and where their SM clocks go
tot = prof[:, 0] + prof[:, 1] + prof[:, 2]
print("slowest entries (start us, duration us, clocks closure/axes/inference, ops, U, depth, rounds, class):")
for i in np.argsort(-end)[:12]:
    print(f"  start {pr[i,0]/1e3:5.1f} dur {pr[i,1]/1e3:5.1f} clocks {prof[i,0]:6d} (descriptor reads {prof[i,7]:5d})/{prof[i,1]:6d}/{prof[i,2]:6d}"
          f" ops {prof[i,3]} U {prof[i,4]} depth {prof[i,5]} rounds {prof[i,6]} class {pr[i,2]}")
print("duration vs clocks: ns per clock p50", np.percentile(pr[:, 1] / np.maximum(tot, 1), 50))
print("entries by start time (us) p0/p50/p100:", np.percentile(pr[:, 0] / 1e3, [0, 50, 100]))
