"""Where the cfg5 one-shot host batch spends its time (run with TP_PROFILE_HOST=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_04285_b200 import engine as E, graph as G, models as M

scen = M.scenario_sweep(1000)
pairs = [(G.flatten(s.graph), s.topo) for s in scen]
sw = E.Sweep(pairs, device=0, host_threads=0)
sw.create()
sw.allocate(pinned=True)
sw.execute()
for rep in range(4):
    t0 = time.perf_counter()
    sw.create()
    t1 = time.perf_counter()
    sw.execute()
    t2 = time.perf_counter()
    print(f"create {1e3 * (t1 - t0):.1f} ms, execute {1e3 * (t2 - t1):.1f} ms", flush=True)
print("threads", os.cpu_count())
