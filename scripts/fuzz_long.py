"""Long randomized parity run (evidence, not a test): N random graphs through the one-shot, the
plan and the scratch paths in both pair forms, and random sweeps through the device-resident
batch, every output compared with the oracle by IEEE bit pattern.
  python scripts/fuzz_long.py [N] [seed]"""
import os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import bindings as B
from paper_2301_04285_b200 import abi, engine, fuzz, graph as G

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 2026)
FIELDS = ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes", "edge_cost_s", "edge_volume_bytes",
          "edge_memory_bytes")


def same(a, b, what):
    for k in ("node_base", "edge_base"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), (what, k)
    for k in FIELDS:
        x, y = getattr(a, k), getattr(b, k)
        assert x.shape == y.shape and np.array_equal(x.view(np.uint64), y.view(np.uint64)), (what, k)


ok = err = 0
ok_graphs = []
for i in range(N):
    g, t = fuzz.random_graph(rng, odd_extents=(i % 2 == 0), mixed_element_sizes=(i % 5 == 0))
    f = G.flatten(g)
    ref = B.oracle_build(f, t)
    runs = [lambda: engine.build_cost_tensors(f, t, pair_form=1 + (i % 2)),
            lambda: engine.build_cost_tensors_oneshot(f, t),
            lambda: engine.Plan(f, t).execute_host()]
    run = runs[i % 3]
    if ref.status != 0:
        try:
            run()
            raise SystemExit(f"graph {i}: the reference throws, the engine did not")
        except (abi.TopoplanError, IndexError):
            err += 1
        continue
    same(run(), ref, f"graph {i}")
    ok += 1
    ok_graphs.append((f, t, ref))
print(f"random graphs: {ok} built bit-identical, {err} errors as the reference", flush=True)
for i in range(N // 2):  # planning instances (valid by construction)
    g, t = fuzz.random_planning_instance(rng)
    f = G.flatten(g)
    ref = B.oracle_build(f, t)
    assert ref.status == 0
    got = (engine.build_cost_tensors(f, t, pair_form=1 + (i % 2)) if i % 3 else engine.build_cost_tensors_oneshot(f, t))
    same(got, ref, f"instance {i}")
    ok_graphs.append((f, t, ref))
print(f"planning instances: {N // 2} built bit-identical", flush=True)
# sweeps of the built graphs through the batched device path (every batch mode's default: 5)
for rep in range(3):
    pick = rng.sample(range(len(ok_graphs)), min(300, len(ok_graphs)))
    ds = engine.DeviceSweep([(ok_graphs[j][0], ok_graphs[j][1]) for j in pick], device=0)
    ds.run()
    ds.check_errors()
    for q, j in enumerate(pick):
        got = {k: v.cpu().numpy() for k, v in ds.result(q).items()}
        for k in FIELDS:
            x, y = got[k], getattr(ok_graphs[j][2], k)
            assert np.array_equal(x.view(np.uint64), y.view(np.uint64)), ("sweep", rep, q, k)
    print(f"device sweep {rep}: {len(pick)} scenarios bit-identical", flush=True)
print("fuzz ok")
