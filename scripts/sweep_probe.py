"""Where the cfg5 host batch spends its time (run with TP_PROFILE_HOST=1): the two-call form
(create + execute) and the one-shot pipelined call (Sweep.build); `--cfg4 K` probes the one-shot
call over K cfg4 builds (the bench's pipelined e2e) instead."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_04285_b200 import engine as E, graph as G, models as M

if "--cfg4" in sys.argv:
    k = int(sys.argv[sys.argv.index("--cfg4") + 1])
    flat = G.flatten(M.cfg4()[0])
    pairs = [(flat, M.cfg4(ratio=2 + r)[1]) for r in range(k)]
else:
    scen = M.scenario_sweep(1000)
    pairs = [(G.flatten(s.graph), s.topo) for s in scen]
sw = E.Sweep(pairs, device=0, host_threads=0)
sw.create()  # the output sizes
sw.allocate(pinned=True)
if "--cfg4" not in sys.argv:
    sw.execute()
    for rep in range(3):
        t0 = time.perf_counter()
        sw.create()
        t1 = time.perf_counter()
        sw.execute()
        t2 = time.perf_counter()
        print(f"create {1e3 * (t1 - t0):.1f} ms, execute {1e3 * (t2 - t1):.1f} ms", flush=True)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sw.build()
    t1 = time.perf_counter()
    print(f"one-shot build {1e3 * (t1 - t0):.2f} ms", flush=True)
print("threads", os.cpu_count())
