"""Full cfg4 build time (device, write-flush) and fan-out trace summary."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2301_04285_b200 import engine as E, graph as G, models as M

g, t = M.cfg4()
plan = E.Plan(G.flatten(g), t, device=0)
ne, nn = plan.sizes["num_aux_edges"], plan.sizes["num_aux_nodes"]
dev = torch.device("cuda", 0)
outs = {k: torch.empty(ne, dtype=torch.float64, device=dev) for k in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes")}
outs.update({k: torch.empty(nn, dtype=torch.float64, device=dev) for k in ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes")})
full = E.device_cost_struct(outs)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
s = torch.cuda.Stream()
plan.upload(s.cuda_stream)
ts = []
with torch.cuda.stream(s):
    for i in range(23):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        plan.execute(full, stream=s.cuda_stream)
        b.record(s)
        if i >= 3:
            ts.append((a, b))
torch.cuda.synchronize()
v = sorted(x.elapsed_time(y) * 1e3 for x, y in ts)
plan.set_timeline(True)
with torch.cuda.stream(s):
    for i in range(4):
        flush.zero_()
        plan.execute(full, stream=s.cuda_stream)
pr, it, fo, _, wx = plan.timeline_detail()
q = lambda x: [round(float(np.percentile(x, p)) / 1e3, 1) for p in (0, 50, 90, 100)]
print(f"build {v[len(v)//2]:.1f} us | pairs end {q(pr[:,0]+pr[:,1])} "
      f"rows end {q(it[:,0]+it[:,1])} | fan n={len(fo)} ready {q(fo[:,0]+fo[:,1])} work {q(fo[:,2]-fo[:,1])} end {q(fo[:,0]+fo[:,2])}")
order = np.argsort(fo[:, 0] + fo[:, 1])[-8:]
for i in order:
    print(f"  late range {i}: start {fo[i,0]/1e3:.1f} wait {fo[i,1]/1e3:.1f} dur {fo[i,2]/1e3:.1f}")
order = np.argsort(fo[:, 0])[:5]
for i in order:
    print(f"  early range {i}: start {fo[i,0]/1e3:.1f} wait {fo[i,1]/1e3:.1f} dur {fo[i,2]/1e3:.1f}")
for c in np.unique(pr[:, 2]):
    m = pr[:, 2] == c
    print(f"  class {c}: pairs {m.sum()}, dur us {q(pr[m, 1])}")
pf = plan.timeline_detail()[3]
print("pricing clocks per pair (closure, axes, inference) pct(0,50,90,100):")
for c in np.unique(pr[:, 2]):
    m = pr[:, 2] == c
    print(f"  class {c}: closure {q(pf[m,0])} axes {q(pf[m,1])} infer {q(pf[m,2])} (k-clocks); ops {q(pf[m,3]*1000)} U {q(pf[m,4]*1000)} depth {q(pf[m,5]*1000)} rounds {q(pf[m,6]*1000)}")
slow = np.argsort(pr[:, 1])[-5:]
for i in slow:
    print(f"  slow pair {i} class {pr[i,2]} dur {pr[i,1]/1e3:.1f}us clocks {list(pf[i,:3])} price {pf[i,7]} ops {pf[i,3]} U {pf[i,4]} depth {pf[i,5]} rounds {pf[i,6]}")
wx = wx[:, 0]
print("warp phase-1 exit us pct:", q(wx))
order = np.argsort(fo[:, 0] + fo[:, 2])[-6:]
for i in order:
    print(f"  slowest-ending range {i}: start {fo[i,0]/1e3:.1f} wait {fo[i,1]/1e3:.1f} dur {fo[i,2]/1e3:.1f}")
# node-row and pair start/duration distributions, and the same build without the L2 flush
print("node rows start us", q(it[:, 0]), "dur", q(it[:, 1]))
print("pairs start us", q(pr[:, 0]), "dur", q(pr[:, 1]))
ts2 = []
with torch.cuda.stream(s):
    for i in range(23):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        plan.execute(full, stream=s.cuda_stream)
        b.record(s)
        if i >= 3:
            ts2.append((a, b))
torch.cuda.synchronize()
v2 = sorted(x.elapsed_time(y) * 1e3 for x, y in ts2)
print(f"build without flush (timeline on) {v2[len(v2)//2]:.1f} us")
plan.set_timeline(False)
ts3 = []
with torch.cuda.stream(s):
    for i in range(23):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        plan.execute(full, stream=s.cuda_stream)
        b.record(s)
        if i >= 3:
            ts3.append((a, b))
torch.cuda.synchronize()
v3 = sorted(x.elapsed_time(y) * 1e3 for x, y in ts3)
print(f"build without flush {v3[len(v3)//2]:.1f} us (with flush {v[len(v)//2]:.1f})")
