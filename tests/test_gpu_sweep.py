"""GPU parity of the batch entry points (tp_plan_create_batch /
tp_plan_execute_host_batch) on cfg5's seeded scenario sweep:
every scenario's cost tensors must be bit-identical to a standalone build of
that scenario by the oracle (build_auxiliary_graph, aux_graph.hpp:211-315),
errors must stay attached to their own scenario, and a sweep must be
re-executable in place."""
import random

import numpy as np
import pytest

from golden_util import bits
from oracle import bindings as B
from paper_2301_04285_b200 import abi, engine, graph as G, models as M

pytestmark = pytest.mark.gpu

FIELDS = ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes",
          "edge_cost_s", "edge_volume_bytes", "edge_memory_bytes")
INDEX = ("node_base", "edge_base", "in_degree", "out_degree", "topo_order", "edge_from_op", "edge_to_op")


def same(gpu, ref, tag):
    for k in INDEX:
        np.testing.assert_array_equal(getattr(gpu, k), getattr(ref, k), err_msg=f"{tag} {k}")
    for k in FIELDS:
        a, b = getattr(gpu, k), getattr(ref, k)
        assert a.shape == b.shape, (tag, k)
        assert np.array_equal(bits(a), bits(b)), f"{tag}: {k} differs"


@pytest.fixture(scope="module")
def sweep1000():
    return M.scenario_sweep(1000)


def test_sweep_first_64_vs_oracle(sweep1000):
    scen = sweep1000[:64]
    flats = [G.flatten(s.graph) for s in scen]
    res = engine.build_sweep([(f, s.topo) for f, s in zip(flats, scen)], device=0, host_threads=6)
    for i, (f, s, r) in enumerate(zip(flats, scen, res)):
        same(r, B.oracle_build(f, s.topo), f"scenario {i} ({s.family})")


def test_full_sweep_counts_and_sample(sweep1000):
    """All 1,000 scenarios in one batch: the aux-edge total SURVEY §8d measured
    on the reference (16,957,929), and a seeded sample checked bit-exact."""
    pairs = [(G.flatten(s.graph), s.topo) for s in sweep1000]
    sw = engine.Sweep(pairs, device=0, host_threads=0)
    sw.create()
    sw.allocate(pinned=True)
    sw.execute()
    assert sw.num_aux_edges == 16_957_929
    assert not sw.status.any()
    for i in random.Random(5).sample(range(1000), 40):
        same(sw.results[i], B.oracle_build(*pairs[i]), f"scenario {i}")
    # executing again in place gives identical bits (pooled arenas are reused)
    snap = {k: bits(getattr(sw.results[7], k)).copy() for k in FIELDS}
    for k in FIELDS:
        getattr(sw.results[7], k)[:] = 0
    sw.execute()
    for k in FIELDS:
        assert np.array_equal(bits(getattr(sw.results[7], k)), snap[k]), k
    sw.destroy()


def test_sweep_errors_stay_with_their_scenario():
    a = M.pointwise_op("a", "x", "y", 8, 8)
    b = M.pointwise_op("b", "y", "x", 8, 8)
    cycle = G.ComputationGraph([a, b], [G.GraphEdge("a", "b", "y"), G.GraphEdge("b", "a", "x")])
    indivisible = G.ComputationGraph([M.dense_op("fc", "matmul", "x", 6, 6, 6, "y")], [])
    g1, t1 = M.cfg1()
    g2, t2 = M.cfg2()
    scen = [(g1, t1), (cycle, G.ClusterTopology(1, 2, 60e9, 60e9, 32e9)), (g2, t2),
            (indivisible, G.ClusterTopology(1, 4, 60e9, 60e9, 32e9)), (g1, t1)]
    flats = [(G.flatten(g), t) for g, t in scen]
    sw = engine.Sweep(flats, device=0, host_threads=3)
    sw.create()
    sw.allocate(pinned=False)
    st = sw.execute(raise_errors=False)
    assert st == abi.TP_ERR_TOPOPLAN
    assert sw.status.tolist() == [0, abi.TP_ERR_TOPOPLAN, 0, abi.TP_ERR_TOPOPLAN, 0]
    for i in (0, 2, 4):
        same(sw.results[i], B.oracle_build(*flats[i]), f"scenario {i}")
    with pytest.raises(abi.TopoplanError):
        sw.execute()
    sw.destroy()


def test_sweep_mixes_owned_and_borrowed_arenas():
    """Plans that were uploaded on their own arena keep it inside a batch."""
    g1, t1 = M.cfg1()
    g2, t2 = M.cfg2()
    pairs = [(G.flatten(g1), t1), (G.flatten(g2), t2), (G.flatten(g1), M.ClusterTopology(2, 4, 60e9, 1e9, 32e9))]
    sw = engine.Sweep(pairs, device=0, host_threads=2)
    sw.create()
    sw.lib.tp_plan_upload(sw.handles[1], None)  # scenario 1 owns an arena from here on
    sw.allocate(pinned=False)
    sw.execute()
    for i, (f, t) in enumerate(pairs):
        same(sw.results[i], B.oracle_build(f, t), f"scenario {i}")
    sw.destroy()


def test_host_batch_records_and_minima(sweep1000):
    """tp_plan_execute_host_batch honours every tp_cost_tensors field: the
    AuxEdge records and the solver minima (cond_min rows, pair_min) of every
    scenario equal the oracle's, as tp_plan_execute_host gives them."""
    scen = sweep1000[:24]
    pairs = [(G.flatten(s.graph), s.topo) for s in scen]
    sw = engine.Sweep(pairs, device=0, host_threads=4)
    sw.create()
    sw.allocate(pinned=False, records=True, row_min=True)
    sw.execute()
    for i, (f, t) in enumerate(pairs):
        ref = B.oracle_build(f, t)
        got = sw.results[i]
        same(got, ref, f"scenario {i}")
        for k in ("row_min_cost_s", "row_min_volume_bytes", "edge_pair_min_cost_s", "edge_pair_min_volume_bytes"):
            n = len(getattr(ref, k))
            assert np.array_equal(bits(getattr(got, k)[:n]), bits(getattr(ref, k))), (i, k)
        ne = len(ref.edge_cost_s)
        a, b = got.records[: ne * 40].reshape(-1, 40).copy(), ref.records.reshape(-1, 40).copy()
        a[:, 12:16] = 0
        b[:, 12:16] = 0
        assert np.array_equal(a, b), i
    sw.destroy()


def test_device_sweep_batched_launch_matches_oracle(sweep1000):
    """The device-resident sweep: one persistent launch for all scenarios
    (tp_plan_execute_batch), repeated (the tables alternate parity), matches
    the oracle on every scenario, every time."""
    import torch
    scen = sweep1000[100:220]
    pairs = [(G.flatten(s.graph), s.topo) for s in scen]
    ds = engine.DeviceSweep(pairs, device=0)
    refs = [B.oracle_build(f, t) for f, t in pairs]
    for rep in range(3):
        for v in ds.out.values():
            v.fill_(float("nan"))
        torch.cuda.synchronize()
        ds.run()
        ds.check_errors()
        for i in range(len(pairs)):
            got = {k: v.cpu().numpy() for k, v in ds.result(i).items()}
            for k in FIELDS:
                assert np.array_equal(bits(got[k]), bits(getattr(refs[i], k))), (rep, i, k)
        assert 1 <= ds.launches_per_run() <= 3  # inference pass + one or two build launches


def test_batch_mixes_forms_errors_and_single_executes():
    """A batch with a thread-form plan (pair_form 2), an error plan and a
    cycle; plans executed alone between batches keep their parity state."""
    import torch
    a = M.pointwise_op("a", "x", "y", 8, 8)
    b = M.pointwise_op("b", "y", "x", 8, 8)
    cycle = G.ComputationGraph([a, b], [G.GraphEdge("a", "b", "y"), G.GraphEdge("b", "a", "x")])
    indivisible = G.ComputationGraph([M.dense_op("fc", "matmul", "x", 6, 6, 6, "y")], [])
    g1, t1 = M.cfg1()
    g2, t2 = M.cfg2()
    scen = [(g1, t1), (g2, t2), (cycle, G.ClusterTopology(1, 2, 60e9, 60e9, 32e9)),
            (indivisible, G.ClusterTopology(1, 4, 60e9, 60e9, 32e9)), (g2, M.ClusterTopology(4, 8, 60e9, 1e9, 80e9))]
    pairs = [(G.flatten(g), t) for g, t in scen]
    ds = engine.DeviceSweep(pairs, device=0)
    ds.plans[1].set_pair_form(2)
    refs = [B.oracle_build(f, t) for f, t in pairs]
    for rep in range(3):
        if rep == 1:  # a plan run alone in between
            ds.plans[4].execute(engine.device_cost_struct(ds.result(4)), stream=ds.main.cuda_stream)
        ds.run()
        torch.cuda.synchronize()
        for i in (0, 1, 4):
            ds.plans[i].check_errors()
            got = {k: v.cpu().numpy() for k, v in ds.result(i).items()}
            for k in FIELDS:
                assert np.array_equal(bits(got[k]), bits(getattr(refs[i], k))), (rep, i, k)
        for i in (2, 3):
            with pytest.raises(abi.TopoplanError):
                ds.plans[i].check_errors()


def test_batch_entry_edge_cases():
    """Empty and single-plan batches; a batch of identical scenarios under
    different bandwidths (one bandwidth group) matches the oracle per member."""
    import ctypes as C
    lib = abi.load_engine()
    assert lib.tp_plan_execute_batch(None, 0, None, None) == abi.TP_OK
    assert lib.tp_plan_execute_host_batch(None, 0, None, None, 0, None) == abi.TP_OK
    g, t = M.cfg2()
    one = engine.build_sweep([(G.flatten(g), t)], device=0)
    same(one[0], B.oracle_build(G.flatten(g), t), "single")
    f = G.flatten(g)
    pairs = [(f, M.ClusterTopology(4, 8, 60e9, 60e9 / r, 80e9)) for r in (1, 2, 3, 5, 7, 10, 20, 50, 100, 150)]
    res = engine.build_sweep(pairs, device=0, host_threads=4)
    for i, (ff, tt) in enumerate(pairs):
        same(res[i], B.oracle_build(ff, tt), f"ratio {i}")


def test_full_sweep_every_scenario_vs_oracle(sweep1000):
    """cfg5 in full: all 1,000 scenarios (16,957,929 aux edges) of the batched
    build, bandwidth groups included, bit-identical to the oracle's standalone
    build of each scenario (oracle builds on a host thread pool)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    pairs = [(G.flatten(s.graph), s.topo) for s in sweep1000]
    sw = engine.Sweep(pairs, device=0, host_threads=0)
    sw.create()
    sw.allocate(pinned=False)
    sw.execute()
    B.oracle()  # load once before the pool
    with ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 1))) as ex:
        refs = list(ex.map(lambda p: B.oracle_build(p[0], p[1], records=False), pairs))
    for i, r in enumerate(refs):
        same(sw.results[i], r, f"scenario {i}")
    sw.destroy()


MODE_CHECK = r"""
import sys, random
sys.path.insert(0, {repo!r})
import numpy as np
from oracle import bindings as B
from paper_2301_04285_b200 import engine, graph as G, models as M
scen = M.scenario_sweep(300)
pairs = [(G.flatten(s.graph), s.topo) for s in scen]
ds = engine.DeviceSweep(pairs, device=0)
for rep in range(2):
    ds.run()
    ds.check_errors()
for i in random.Random(3).sample(range(300), 25):
    got = {{k: v.cpu().numpy() for k, v in ds.result(i).items()}}
    ref = B.oracle_build(*pairs[i])
    for k, v in got.items():
        assert np.array_equal(v.view(np.uint64), getattr(ref, k).view(np.uint64)), (i, k)
sw = engine.Sweep(pairs[:60], device=0, host_threads=4)
sw.create(); sw.allocate(pinned=True); sw.execute()
for i in range(0, 60, 7):
    ref = B.oracle_build(*pairs[i])
    for k in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes", "node_intra_cost_s"):
        assert np.array_equal(getattr(sw.results[i], k).view(np.uint64), getattr(ref, k).view(np.uint64)), (i, k)
print("mode ok", ds.launches_per_run())
"""


@pytest.mark.parametrize("mode", ["0", "4", "5"])
def test_batch_modes_match_oracle(mode):
    """Every batch mode (TP_BATCH_MODE: 0 = class tables published in one
    launch, 4 = priced in the fan-out from op lists, 5 = tables from op lists
    in a launch of their own) gives the oracle's bits, device-resident and
    through the host batch."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TP_BATCH_MODE=mode)
    r = subprocess.run([sys.executable, "-c", MODE_CHECK.format(repo=repo)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "mode ok" in r.stdout


def test_one_shot_pipelined_sweep(sweep1000):
    """tp_build_cost_tensors_batch: analysis and build pipelined in chunks,
    kernels writing the pinned slices directly -- every scenario's tensors
    equal the oracle's; pageable slices (staged) too; errors per scenario."""
    scen = sweep1000[:300]
    pairs = [(G.flatten(s.graph), s.topo) for s in scen]
    for pinned in (True, False):
        sw = engine.Sweep(pairs, device=0, host_threads=4)
        sw.create()
        sw.allocate(pinned=pinned)
        sw.destroy()  # build() analyses on its own
        for k in FIELDS:
            for r in sw.results:
                getattr(r, k)[:] = np.nan
        sw.build()
        assert not sw.status.any()
        for i in list(range(0, 300, 23)) + [299]:
            same(sw.results[i], B.oracle_build(*pairs[i]), f"scenario {i} pinned={pinned}")
    a = M.pointwise_op("a", "x", "y", 8, 8)
    b = M.pointwise_op("b", "y", "x", 8, 8)
    cycle = G.ComputationGraph([a, b], [G.GraphEdge("a", "b", "y"), G.GraphEdge("b", "a", "x")])
    g1, t1 = M.cfg1()
    mixed = [(G.flatten(g1), t1), (G.flatten(cycle), G.ClusterTopology(1, 2, 60e9, 60e9, 32e9))] + pairs[:200]
    sw = engine.Sweep(mixed, device=0, host_threads=4)
    sw.create(raise_errors=False)
    sw.allocate(pinned=True)
    st = sw.build(raise_errors=False)
    assert st == abi.TP_ERR_TOPOPLAN
    assert sw.status[1] == abi.TP_ERR_TOPOPLAN and sw.status[0] == 0 and not sw.status[2:].any()
    same(sw.results[0], B.oracle_build(*mixed[0]), "cfg1 beside a cycle")
    same(sw.results[150], B.oracle_build(*mixed[150]), "scenario 148 beside a cycle")
