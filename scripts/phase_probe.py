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

for form in (1, 2):
    plan.set_pair_form(form)
    plan.set_timeline(True)
    for kw in ({}, {"edge_range": (0, 0)}):
        tl = []
        with torch.cuda.stream(s):
            for i in range(8):
                flush.zero_()
                plan.execute(full, stream=s.cuda_stream, **kw)
                tl.append(plan.timeline())
        tl = tl[3:]
        med = {k: sorted(t[k] for t in tl)[len(tl) // 2] / 1e3 for k in tl[0]}
        print(f"form {form} {kw or 'full'} timeline us:", {k: round(v, 1) for k, v in med.items()})
    plan.set_timeline(False)

import numpy as np
print("sizes", plan.sizes)
for form in (1, 2):
    plan.set_pair_form(form)
    plan.set_timeline(True)
    with torch.cuda.stream(s):
        for i in range(4):
            flush.zero_()
            plan.execute(full, stream=s.cuda_stream)
    pr, it, fo, _, _ = plan.timeline_detail()
    q = lambda v: [round(float(np.percentile(v, x)) / 1e3, 2) for x in (0, 10, 50, 90, 99, 100)] if len(v) else []
    print(f"form {form} pair dur us pct(0,10,50,90,99,100):", q(pr[:, 1]), "sum ms", pr[:, 1].sum() / 1e6)
    print(f"form {form} pair start us pct:", q(pr[:, 0]), " end:", q(pr[:, 0] + pr[:, 1]))
    print(f"form {form} row dur us pct:", q(it[:, 1]), "end:", q(it[:, 0] + it[:, 1]), "n", len(it))
    print(f"form {form} fan-out n {len(fo)} start:", q(fo[:, 0]), "wait:", q(fo[:, 1]), "dur:", q(fo[:, 2]),
          "end:", q(fo[:, 0] + fo[:, 2]))
    if form == 1:
        np.save("gpurun_out/pair_ns.npy", pr)
    plan.set_timeline(False)

# speed of light for the fan-out stores in the bench's setting: zero the three
# edge arrays (51.7 MB) after a write flush / after a read flush
rd = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
def t_store(read_flush, n=20, fn=None):
    ts = []
    with torch.cuda.stream(s):
        for i in range(n + 3):
            flush.zero_()
            if read_flush:
                rd.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            if fn is None:
                for k in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes"):
                    outs[k].zero_()
            else:
                fn()
            b.record(s)
            if i >= 3:
                ts.append((a, b))
    torch.cuda.synchronize()
    v = sorted(x.elapsed_time(y) * 1e3 for x, y in ts)
    return v[len(v) // 2]
plan.set_pair_form(1)
print(f"zero 3 edge arrays: write-flush {t_store(False):.1f} us, read-flush {t_store(True):.1f} us")
print(f"full build: write-flush {t_store(False, fn=lambda: plan.execute(full, stream=s.cuda_stream)):.1f} us, "
      f"read-flush {t_store(True, fn=lambda: plan.execute(full, stream=s.cuda_stream)):.1f} us")
big = torch.empty(3 * ne, dtype=torch.float64, device=dev)
print(f"zero one 51.7MB array: write-flush {t_store(False, fn=lambda: big.zero_()):.1f} us")
