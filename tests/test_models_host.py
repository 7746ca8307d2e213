"""Host-side logic: model builders vs the reference's models.hpp, the
benchmark configurations' sizes, graph validation
(graph.hpp:201-351) and the flattened descriptor."""
import ctypes as C
import json

import pytest

from oracle import bindings as B
from paper_2301_04285_b200 import graph as G, models as M


def ref_model(spec):
    lib = B.reference()
    n = lib.ref_model_json(spec.encode(), None, 0)
    buf = C.create_string_buffer(n + 1)
    lib.ref_model_json(spec.encode(), buf, n + 1)
    return json.loads(buf.value.decode())


def as_json(g):
    return {"operators": [{"id": o.id, "kind": o.kind,
                           "inputs": [{"name": t.name, "shape": list(t.shape), "element_size": t.element_size}
                                      for t in o.inputs],
                           "outputs": [{"name": t.name, "shape": list(t.shape), "element_size": t.element_size}
                                       for t in o.outputs],
                           "axes": [{"name": a.name, "slices": [{"tensor": s.tensor, "dim": s.dim} for s in a.slices]}
                                    for a in o.axes]} for o in g.operators],
            "edges": [{"from": e.from_, "to": e.to, "tensor": e.tensor} for e in g.edges]}


@pytest.mark.skipif(not B.have_reference(), reason="oracle/_ref not built")
@pytest.mark.parametrize("spec", ["mlp-chain", "mlp-chain:layers=5,hidden=512,batch=32", "transformer-layer",
                                  "transformer-layer:hidden=4096,batch=8,seq=512", "alexnet-like",
                                  "alexnet-like:batch=16"])
def test_builders_match_reference(spec):
    assert as_json(M.build_graph(M.parse_model_spec(spec))) == ref_model(spec)


def sizes(g, t):
    return B.sizes(G.flatten(g), t)


def test_config_sizes():
    assert sizes(*M.cfg1())[:2] == (48, 252)
    assert sizes(*M.cfg2())[:2] == (438, 7860)
    assert sizes(*M.cfg3(2))[:2] == (6768, 95936)
    assert sizes(*M.cfg3(4))[:2] == (10512, 190940)
    assert sizes(*M.cfg3(8))[:2] == (15120, 335088)
    assert sizes(*M.cfg4())[:2] == (82368, 2155580)


def test_cfg5_scenario_sweep_total():
    """1,000 seeded scenarios; SURVEY.md §8d measured 16,957,929 evals."""
    total = 0
    for s in M.scenario_sweep(1000):
        r = sizes(s.graph, s.topo)
        total += r[1]
    assert total == 16957929


def test_gpt_chain_is_valid():
    g = M.build_gpt_chain(3, 256, 2, 16)
    assert G.validate_graph(g).ok()
    assert len(g.operators) == 36 and len(g.edges) == 3 * 15 + 2


def test_validation_codes():  # test_graph.cpp analogues
    g, _ = M.cfg1()
    assert G.validate_graph(g).ok()
    bad = G.ComputationGraph([M.pointwise_op("a", "x", "y", 8, 8), M.pointwise_op("a", "y", "z", 8, 8)],
                             [G.GraphEdge("a", "b", "y")])
    r = G.validate_graph(bad)
    assert r.has("duplicate-id") and r.has("dangling-reference")
    cyc = G.ComputationGraph([M.pointwise_op("a", "x", "y", 8, 8), M.pointwise_op("b", "y", "x", 8, 8)],
                             [G.GraphEdge("a", "b", "y"), G.GraphEdge("b", "a", "x")])
    assert G.validate_graph(cyc).has("cycle")
    assert G.validate_topology(G.ClusterTopology(1, 3, 60e9, 6e9, 1e9)).has("power-of-two")
    assert not G.validate_topology(G.ClusterTopology(2, 8, 60e9, 6e9, 32e9)).issues
    assert G.validate_topology(G.ClusterTopology(2, 8, 6e9, 60e9, 32e9)).has("bandwidth-order")


def test_flatten_interns_names():
    g, _ = M.cfg1()
    f = G.flatten(g)
    assert f.num_ops == 3 and f.num_edges == 2
    assert list(f.op_tensor_begin) == [0, 3, 5, 8]
    assert list(f.op_axis_begin) == [0, 3, 5, 8]
    assert f.names["x1"] == f.edge_tensor[0]


def composer_json(which, a, b, c=0, d=0):
    lib = B.reference()
    n = lib.ref_composer_json(which, a, b, c, d, None, 0)
    assert n >= 0, lib.ref_last_error()
    buf = C.create_string_buffer(n + 1)
    lib.ref_composer_json(which, a, b, c, d, buf, n + 1)
    return json.loads(buf.value.decode())


@pytest.mark.skipif(not B.have_reference(), reason="oracle/_ref not built")
def test_cpp_composer_matches_python():
    """include/taps_b200/models_b200.hpp (the C++ callers' composer) builds the
    same GPT chains and the same cfg5 scenarios as models.py."""
    assert composer_json(0, 3, 256, 2, 16) == as_json(M.build_gpt_chain(3, 256, 2, 16))
    sweep = M.scenario_sweep(1000)
    for i in (0, 1, 2, 3, 5, 8, 13, 21, 34, 55, 89, 144, 233, 377, 610, 987, 999):
        j = composer_json(1, i, 1000)
        s = sweep[i]
        assert j["graph"] == as_json(s.graph), i
        t = s.topo
        assert j["topo"] == [t.node_count, t.local_device_num, t.intra_bandwidth, t.inter_bandwidth, t.device_memory]
