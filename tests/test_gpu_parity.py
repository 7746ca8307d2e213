"""GPU parity: the CUDA engine (through its C-ABI) against the oracle and the
reference's golden vectors. Bit-exact for every integer/index output and for
the fp64 costs (the north star allows 1e-6 relative; the kernels keep the
reference's operation order, so we hold them to identical bits)."""
import random

import numpy as np
import pytest

from golden_util import bits, golden, graph_of, topo_of, unhex
from oracle import bindings as B
from paper_2301_04285_b200 import abi, engine, fuzz, graph as G, models as M

pytestmark = pytest.mark.gpu

FIELDS = ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes",
          "edge_cost_s", "edge_volume_bytes", "edge_memory_bytes")
INDEX = ("node_base", "edge_base", "in_degree", "out_degree", "topo_order", "edge_from_op", "edge_to_op")


def gpu_build(g, t, **kw):
    return engine.build_cost_tensors(g, t, **kw)


FORMS = [1, 2]  # pair path: warp per pair, thread per pair


def assert_same(gpu, ref, rowmin=False, records=False):
    for k in INDEX:
        np.testing.assert_array_equal(getattr(gpu, k), getattr(ref, k), err_msg=k)
    for k in FIELDS:
        a, b = getattr(gpu, k), getattr(ref, k)
        assert a.shape == b.shape, k
        bad = np.flatnonzero(bits(a) != bits(b))
        assert bad.size == 0, f"{k}: {bad.size} mismatches, first {bad[:5]} gpu={a[bad[:3]]} ref={b[bad[:3]]}"
    if rowmin:
        for k in ("row_min_cost_s", "row_min_volume_bytes", "edge_pair_min_cost_s", "edge_pair_min_volume_bytes"):
            assert np.array_equal(bits(getattr(gpu, k)), bits(getattr(ref, k))), k
    if records:
        ra = gpu.records.reshape(-1, 40).copy()
        rb = ref.records.reshape(-1, 40).copy()
        ra[:, 12:16] = 0  # AuxEdge padding (uninitialised in the reference)
        rb[:, 12:16] = 0
        assert np.array_equal(ra, rb)


def test_abi_version(engine):
    assert engine.tp_abi_version() == abi.TP_ABI_VERSION == 2


@pytest.mark.parametrize("p,N", [(1, 1), (2, 8), (3, 4), (3, 8), (2, 128), (3, 128), (4, 64), (5, 32)])
def test_strategy_tables_match_oracle(p, N):
    got = engine.enumerate_strategies(p, N)
    exp = B.enumerate_with(B.oracle().oracle_enumerate, p, N)
    for a, b in zip(got, exp):
        np.testing.assert_array_equal(a, b)


def test_strategy_tables_golden():
    for tab in golden()["strategy_tables"]:
        deg, dm, md, dep = engine.enumerate_strategies(tab["p"], tab["N"])
        assert deg.tolist() == tab["degrees"]
        assert dm.tolist() == tab["device_map"]
        assert md.tolist() == tab["matrix"]
        assert dep.tolist() == tab["depth"]


def test_table3_rows():
    """The nine MatMul strategies on four devices (test_layout.cpp:67-99)."""
    deg, dm, md, dep = engine.enumerate_strategies(3, 4)
    assert deg.tolist() == [[1, 1, 4], [1, 2, 2], [1, 2, 2], [1, 4, 1], [2, 1, 2], [2, 1, 2], [2, 2, 1],
                            [2, 2, 1], [4, 1, 1]]
    assert dm.tolist() == [[-1, -1, 0], [-1, 1, 0], [-1, 0, 1], [-1, 0, -1], [1, -1, 0], [0, -1, 1],
                           [1, 0, -1], [0, 1, -1], [0, -1, -1]]


def _query(c):
    return B.make_query(c["shape"], c["from_dims"], c["from_map"], c["to_dims"], c["to_map"],
                        tensor_bytes=c["tensor_bytes"], local=c["local"], intra=c["intra"], inter=c["inter"])


@pytest.mark.parametrize("form", FORMS)
def test_redistribution_goldens(form):
    cases = golden()["redistributions"]
    qs = [_query(c) for c in cases]
    res = engine.redistribute_batch(qs, form=form)
    for c, r in zip(cases, res):
        if c["status"] != 0:
            assert r.status != 0, c
            continue
        assert r.status == 0, (c, r.status)
        dims, ushape, ufm, utm, ops, cts = r.plan()
        assert list(dims) == c["dims"]
        assert list(ushape) == c["ushape"]
        assert list(ufm) == c["ufrom"] and list(utm) == c["uto"]
        assert [list(o) for o in ops] == c["ops"]
        assert list(cts) == c["ct"]
        assert np.array_equal(bits(r.op_seconds[: r.num_ops]), bits(unhex(c["op_seconds"])))
        assert bits([r.volume_bytes])[0] == bits([unhex(c["volume"])])[0]
        assert bits([r.seconds])[0] == bits([unhex(c["seconds"])])[0]


@pytest.mark.parametrize("form", FORMS)
def test_redistribution_random_vs_oracle(form):
    rng = random.Random(99)
    qs = []
    for i in range(4000):
        dims, shape, fm, tm = fuzz.random_redist_case(rng)
        if i % 2:
            d2 = fuzz.random_matrix_with_total(rng, int(np.prod(dims)))
            tm = fuzz.random_map_for(rng, shape, d2)
        else:
            d2 = dims
        if i % 3 == 0:
            shape = [s * rng.choice([1, 3, 5, 7]) for s in shape]
        qs.append(B.make_query(shape, dims, fm, d2, tm, local=rng.choice([1, 2, 4, 8, 16]),
                               inter=rng.choice([6e9, 60e9, 1.5e9])))
    res = engine.redistribute_batch(qs, form=form)
    for q, r in zip(qs, res):
        o = B.oracle_redistribute(q)
        assert r.status == o.status
        if o.status == 0:
            assert r.plan() == o.plan()
            assert bits([r.seconds])[0] == bits([o.seconds])[0]
            assert bits([r.volume_bytes])[0] == bits([o.volume_bytes])[0]


@pytest.mark.parametrize("form", FORMS)
@pytest.mark.parametrize("idx", range(len(golden()["builds"])))
def test_golden_builds(idx, form):
    c = golden()["builds"][idx]
    g, t = graph_of(c["graph"]), topo_of(c["topo"])
    got = gpu_build(g, t, row_min=True, pair_form=form)
    assert got.node_base.tolist() == c["node_base"]
    assert got.edge_base.tolist() == c["edge_base"]
    assert got.topo_order.tolist() == c["topo_order"]
    for k in FIELDS + ("row_min_cost_s", "row_min_volume_bytes", "edge_pair_min_cost_s", "edge_pair_min_volume_bytes"):
        exp = unhex(c[k])
        assert np.array_equal(bits(getattr(got, k)), bits(exp)), (c["name"], k)


@pytest.mark.parametrize("form", FORMS)
@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_configs_vs_oracle(name, form):
    g, t = M.CONFIGS[name]()
    f = G.flatten(g)
    gpu = gpu_build(f, t, records=True, row_min=True, pair_form=form)
    ref = B.oracle_build(f, t)
    assert ref.status == 0
    assert_same(gpu, ref, rowmin=True, records=True)
    if name == "cfg1":
        assert len(gpu.node_intra_cost_s) == 48 and len(gpu.edge_cost_s) == 252


@pytest.mark.parametrize("form", FORMS)
@pytest.mark.parametrize("nodes,ratio", [(2, 1), (4, 10), (8, 100)])
def test_cfg3_vs_oracle(nodes, ratio, form):
    g, t = M.cfg3(nodes, ratio)
    f = G.flatten(g)
    gpu = gpu_build(f, t, pair_form=form)
    ref = B.oracle_build(f, t, records=False)
    assert_same(gpu, ref)
    assert len(gpu.edge_cost_s) == {2: 95936, 4: 190940, 8: 335088}[nodes]


@pytest.mark.parametrize("form", FORMS)
@pytest.mark.parametrize("ratio", [10, 100])
def test_cfg4_vs_oracle(ratio, form):
    """cfg4 (GPT-96, hidden 12288, 16x8; the bench workload) in full: every
    one of the 2,155,580 aux edges and 82,368 aux nodes bit-identical."""
    g, t = M.cfg4(ratio)
    f = G.flatten(g)
    gpu = gpu_build(f, t, row_min=True, pair_form=form)
    ref = B.oracle_build(f, t, records=False)
    assert ref.status == 0
    assert_same(gpu, ref, rowmin=True)
    assert len(gpu.edge_cost_s) == 2155580 and len(gpu.node_intra_cost_s) == 82368


@pytest.mark.parametrize("form", FORMS)
def test_random_graphs_vs_oracle(form):
    rng = random.Random(1234)
    ok = err = 0
    for i in range(150):
        g, t = fuzz.random_graph(rng, odd_extents=(i % 2 == 0), mixed_element_sizes=(i % 5 == 0))
        f = G.flatten(g)
        ref = B.oracle_build(f, t)
        if ref.status != 0:
            with pytest.raises((abi.TopoplanError, IndexError)):
                gpu_build(f, t, pair_form=form)
            err += 1
            continue
        gpu = gpu_build(f, t, records=True, row_min=True, pair_form=form)
        assert_same(gpu, ref, rowmin=True, records=True)
        ok += 1
    assert ok > 20 and err > 10


@pytest.mark.parametrize("form", FORMS)
def test_planning_instances_vs_oracle(form):
    rng = random.Random(17)
    for _ in range(40):
        g, t = fuzz.random_planning_instance(rng)
        f = G.flatten(g)
        assert_same(gpu_build(f, t, row_min=True, pair_form=form), B.oracle_build(f, t), rowmin=True)


def test_edge_range_shards_concatenate():
    g, t = M.cfg2()
    f = G.flatten(g)
    full = gpu_build(f, t)
    plan = engine.Plan(f, t)
    cuts = [0, 4, 9, 15]
    parts = [plan.execute_host(edge_range=(a, b)) for a, b in zip(cuts[:-1], cuts[1:])]
    for k in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes"):
        cat = np.concatenate([getattr(p, k) for p in parts])
        assert np.array_equal(bits(cat), bits(getattr(full, k)))


def test_errors_match_reference_class():
    # indivisible extent (test_aux_graph.cpp:216-220)
    g = G.ComputationGraph([M.dense_op("fc", "matmul", "x", 6, 6, 6, "y")], [])
    with pytest.raises(abi.TopoplanError):
        gpu_build(g, G.ClusterTopology(1, 4, 60e9, 60e9, 32e9))
    # non power-of-two device count
    with pytest.raises(abi.TopoplanError):
        gpu_build(g, G.ClusterTopology(3, 1, 60e9, 60e9, 32e9))
    # cycle
    a = M.pointwise_op("a", "x", "y", 8, 8)
    b = M.pointwise_op("b", "y", "x", 8, 8)
    with pytest.raises(abi.TopoplanError):
        gpu_build(G.ComputationGraph([a, b], [G.GraphEdge("a", "b", "y"), G.GraphEdge("b", "a", "x")]),
                  G.ClusterTopology(1, 2, 60e9, 60e9, 32e9))
    # edge tensor absent from the producer -> std::out_of_range
    with pytest.raises(IndexError):
        gpu_build(G.ComputationGraph([a, M.pointwise_op("c", "y", "z", 8, 8)], [G.GraphEdge("a", "c", "q")]),
                  G.ClusterTopology(1, 2, 60e9, 60e9, 32e9))
    # dangling edge
    with pytest.raises(abi.TopoplanError):
        gpu_build(G.ComputationGraph([a], [G.GraphEdge("a", "nope", "y")]), G.ClusterTopology(1, 2, 60e9, 60e9, 32e9))


def test_single_device_and_empty():
    g = G.ComputationGraph([M.dense_op("fc", "matmul", "x", 8, 8, 8, "y")], [])
    r = gpu_build(g, G.ClusterTopology(1, 1, 60e9, 60e9, 32e9))
    assert r.node_intra_cost_s.tolist() == [0.0] and r.node_intra_volume_bytes.tolist() == [0.0]
    e = gpu_build(G.ComputationGraph([], []), G.ClusterTopology(1, 8, 60e9, 6e9, 32e9))
    assert len(e.edge_cost_s) == 0 and len(e.node_intra_cost_s) == 0


def test_shared_layouts_and_derived_classes():
    """Class tables over distinct layouts (and classes derived by an exact
    power-of-two byte ratio) are bit-exact, and they do shrink the pair work:
    some random graphs price fewer entries than their classes' strategy pairs."""
    rng = random.Random(99)
    shrunk = 0
    for i in range(60):
        g, t = fuzz.random_graph(rng, odd_extents=False, mixed_element_sizes=(i % 3 == 0))
        f = G.flatten(g)
        ref = B.oracle_build(f, t)
        if ref.status != 0:
            continue
        plan = engine.Plan(f, t, device=0)
        sz = plan.sizes
        assert sz["num_pair_evals"] <= sz["num_pair_slots"]
        shrunk += sz["num_pair_evals"] < sz["num_pair_slots"]
        del plan
        assert_same(gpu_build(f, t, row_min=True), ref, rowmin=True)
    g, t = M.cfg4()
    sz = engine.Plan(G.flatten(g), t, device=0).sizes
    assert sz["num_pair_evals"] < sz["num_pair_slots"] * 0.55  # GPT: the 4h-wide classes derive from the h-wide ones
    assert shrunk > 0


def test_timeline_diagnostics():
    import torch
    g, t = M.cfg2()
    f = G.flatten(g)
    plan = engine.Plan(f, t, device=0)
    sz = plan.sizes
    dev = torch.device("cuda", 0)
    outs = {k: torch.empty(sz["num_aux_edges"], dtype=torch.float64, device=dev)
            for k in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes")}
    outs.update({k: torch.empty(sz["num_aux_nodes"], dtype=torch.float64, device=dev)
                 for k in ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes")})
    plan.set_timeline(True)
    plan.execute(engine.device_cost_struct(outs))
    tl = plan.timeline()
    assert tl["end"] > 0 and tl["first_fanout"] > 0
    pairs, rows, ranges, clocks, exits = plan.timeline_detail()
    assert pairs.shape == (sz["num_pair_evals"], 3) and (pairs[:, 1] > 0).all()
    assert rows.shape == (sz["num_class_rows"], 2) and (rows[:, 1] > 0).all()
    assert ranges.shape[1] == 3 and (ranges[:, 2] > 0).all()
    assert clocks.shape == (sz["num_pair_evals"], 8)
    assert exits.shape[1] == 1 and exits.shape[0] % 8 == 0
    plan.set_timeline(False)
    plan.execute(engine.device_cost_struct(outs))
    plan.check_errors()
    ref = B.oracle_build(f, t)
    np.testing.assert_array_equal(bits(outs["edge_cost_s"].cpu().numpy()), bits(ref.edge_cost_s))


@pytest.mark.parametrize("nodes", [2, 8])
def test_cfg3_ratio_sweep_by_repricing(nodes):
    """cfg3's sweep of the intra/inter bandwidth ratio (1, 2, 5,
    10, 20, 50, 100 with intra 60 GB/s) on ONE analysed plan re-priced with
    tp_plan_set_bandwidth: every ratio bit-identical to a fresh oracle build."""
    g, _ = M.cfg3(nodes, 10)
    f = G.flatten(g)
    plan = engine.Plan(f, M.cfg3(nodes, 10)[1], device=0)
    for ratio in (10, 1, 2, 5, 20, 50, 100):
        t = M.cfg3(nodes, ratio)[1]
        plan.set_bandwidth(t.intra_bandwidth, t.inter_bandwidth)
        got = plan.execute_host(row_min=True)
        ref = B.oracle_build(f, t, records=False)
        assert_same(got, ref, rowmin=True)


def test_pair_min_device_and_slices():
    """pair_min (solver.hpp:254-255) on device tensors and on edge slices, bit-identical to the
    oracle (itself pinned to the reference's make_context); pair outputs without the row minima
    are rejected with TP_ERR_INVALID_ARGUMENT before any launch."""
    import torch
    from paper_2301_04285_b200 import abi
    g, t = M.cfg2()
    f = G.flatten(g)
    ref = B.oracle_build(f, t, records=False)
    plan = engine.Plan(f, t, device=0)
    sz = plan.sizes
    dev = torch.device("cuda", 0)
    ne, nr = f.num_edges, int(sz["num_rows"])
    outs = {k: torch.empty(sz["num_aux_edges"], dtype=torch.float64, device=dev)
            for k in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes")}
    outs["edge_pair_min_cost_s"] = torch.empty(ne, dtype=torch.float64, device=dev)
    outs["edge_pair_min_volume_bytes"] = torch.empty(ne, dtype=torch.float64, device=dev)
    with pytest.raises(ValueError):
        plan.execute(engine.device_cost_struct(outs))
    outs["row_min_cost_s"] = torch.empty(nr, dtype=torch.float64, device=dev)
    outs["row_min_volume_bytes"] = torch.empty(nr, dtype=torch.float64, device=dev)
    plan.execute(engine.device_cost_struct(outs))
    plan.check_errors()
    for k in ("row_min_cost_s", "row_min_volume_bytes", "edge_pair_min_cost_s", "edge_pair_min_volume_bytes"):
        assert np.array_equal(bits(outs[k].cpu().numpy()), bits(getattr(ref, k))), k
    for e0, e1 in ((0, 1), (3, 9), (ne - 2, ne)):
        got = plan.execute_host(row_min=True, edge_range=(e0, e1))
        np.testing.assert_array_equal(bits(got.edge_pair_min_cost_s), bits(ref.edge_pair_min_cost_s[e0:e1]))
        np.testing.assert_array_equal(bits(got.edge_pair_min_volume_bytes),
                                      bits(ref.edge_pair_min_volume_bytes[e0:e1]))


def test_cfg4_minima_properties():
    """Full cfg4 (2,155,580 aux edges): the device row and pair minima equal
    the minima of the device's own cost blocks (solver.hpp:239-255), both
    modes — a size-independent check next to the oracle comparisons."""
    g, t = M.cfg4()
    ct = gpu_build(g, t, row_min=True)
    nb, eb = ct.node_base, ct.edge_base
    r = 0
    for e in range(len(ct.edge_from_op)):
        su_n = int(nb[ct.edge_from_op[e] + 1] - nb[ct.edge_from_op[e]])
        sw_n = int(nb[ct.edge_to_op[e] + 1] - nb[ct.edge_to_op[e]])
        for src, rows, pair in (("edge_cost_s", "row_min_cost_s", "edge_pair_min_cost_s"),
                                ("edge_volume_bytes", "row_min_volume_bytes", "edge_pair_min_volume_bytes")):
            blk = getattr(ct, src)[eb[e]:eb[e] + su_n * sw_n].reshape(su_n, sw_n)
            rm = blk.min(axis=1)
            assert np.array_equal(bits(rm), bits(getattr(ct, rows)[r:r + su_n])), (e, rows)
            assert bits(np.array([rm.min()]))[0] == bits(getattr(ct, pair)[e:e + 1])[0], (e, pair)
        r += su_n
    assert r == len(ct.row_min_cost_s)


PAR_CHECK = r"""
import random, sys
sys.path.insert(0, {repo!r}); sys.path.insert(0, {repo!r} + "/tests")
import numpy as np
from oracle import bindings as B
from paper_2301_04285_b200 import abi, engine, fuzz, graph as G, models as M
from golden_util import bits
def same(a, b):
    for k in ("node_base", "edge_base", "in_degree", "out_degree", "topo_order", "edge_from_op", "edge_to_op"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    for k in ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes", "edge_cost_s",
              "edge_volume_bytes", "edge_memory_bytes"):
        assert np.array_equal(bits(getattr(a, k)), bits(getattr(b, k))), k
rng = random.Random(99)
n_ok = n_err = 0
for i in range(120):
    g, t = fuzz.random_graph(rng, odd_extents=(i % 2 == 0), mixed_element_sizes=(i % 5 == 0))
    f = G.flatten(g)
    ref = B.oracle_build(f, t)
    if ref.status != 0:
        try:
            engine.build_cost_tensors(f, t)
            raise SystemExit("expected an error at graph %d" % i)
        except (abi.TopoplanError, IndexError):
            n_err += 1
        continue
    same(engine.build_cost_tensors(f, t), ref)
    n_ok += 1
for g, t in (M.cfg2(), M.cfg3(2, 10)):
    f = G.flatten(g)
    same(engine.build_cost_tensors(f, t), B.oracle_build(f, t))
print("par ok", n_ok, n_err)
"""


def test_parallel_host_analysis_matches_oracle():
    """The host analysis's per-op / per-edge passes on the worker pool (forced
    on small graphs, one op or edge per work item) give the oracle's bits and
    the reference's errors."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TP_HOST_PAR_MIN="1", TP_HOST_WORKERS="8")
    r = subprocess.run([sys.executable, "-c", PAR_CHECK.format(repo=repo)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "par ok" in r.stdout


def test_one_shot_and_scratch_calls_match_oracle():
    """tp_build_cost_tensors (the reference-facing one-shot call) and
    tp_plan_execute_host_scratch reuse the calling thread's device memory
    across graphs of different sizes: a sequence of different graphs,
    alternating those two with a plan's own memory, every build bit-identical
    to the oracle and every error the reference's."""
    rng = random.Random(7)
    cases = [M.cfg2(), M.cfg1(), M.cfg3(2, 10)] + [fuzz.random_graph(rng) for _ in range(60)] + [M.cfg2()]
    ok = err = 0
    for i, (g, t) in enumerate(cases):
        f = G.flatten(g)
        ref = B.oracle_build(f, t)
        run = (lambda: engine.build_cost_tensors_oneshot(f, t), lambda: engine.Plan(f, t).execute_host(scratch=True),
               lambda: engine.build_cost_tensors(f, t))[i % 3]
        if ref.status != 0:
            with pytest.raises((abi.TopoplanError, IndexError)):
                run()
            err += 1
            continue
        assert_same(run(), ref)
        ok += 1
    assert ok > 15 and err > 10
    # a plan with device memory of its own keeps using it; scratch calls between its builds
    f, t = G.flatten(M.cfg2()[0]), M.cfg2()[1]
    plan = engine.Plan(f, t)
    ref = B.oracle_build(f, t)
    assert_same(plan.execute_host(), ref)
    assert_same(engine.build_cost_tensors_oneshot(*(G.flatten(M.cfg1()[0]), M.cfg1()[1])),
                B.oracle_build(G.flatten(M.cfg1()[0]), M.cfg1()[1]))
    assert_same(plan.execute_host(scratch=True), ref)
    assert_same(plan.execute_host(), ref)
