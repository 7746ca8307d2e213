"""Generates the golden fixtures of tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/libtopoplan_ref.so, compiled from /root/reference by
oracle/Makefile). Run here, where the reference exists:

    python tests/golden/make_golden.py

Doubles are stored as IEEE-754 hex strings so comparisons are bit-exact.
"""
import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import bindings as B  # noqa: E402
from paper_2301_04285_b200 import graph as G, models as M, fuzz  # noqa: E402


def hx(a):
    return [struct.pack("<d", float(x)).hex() for x in np.asarray(a, dtype=np.float64)]


def build_case(name, g, t, solve=False, threads=8):
    f = G.flatten(g)
    r = B.reference_build(f, t)
    case = dict(name=name, graph=graph_json(g), topo=dict(node_count=t.node_count, local_device_num=t.local_device_num,
                intra_bandwidth=t.intra_bandwidth, inter_bandwidth=t.inter_bandwidth, device_memory=t.device_memory),
                status=int(r.status))
    if r.status == 0:
        case.update(node_base=r.node_base.tolist(), edge_base=r.edge_base.tolist(),
                    in_degree=r.in_degree.tolist(), out_degree=r.out_degree.tolist(), topo_order=r.topo_order.tolist(),
                    node_intra_cost_s=hx(r.node_intra_cost_s), node_intra_volume_bytes=hx(r.node_intra_volume_bytes),
                    node_memory_bytes=hx(r.node_memory_bytes), edge_cost_s=hx(r.edge_cost_s),
                    edge_volume_bytes=hx(r.edge_volume_bytes), edge_memory_bytes=hx(r.edge_memory_bytes),
                    row_min_cost_s=hx(r.row_min_cost_s), row_min_volume_bytes=hx(r.row_min_volume_bytes),
                    edge_pair_min_cost_s=hx(r.edge_pair_min_cost_s),  # make_context's pair_min
                    edge_pair_min_volume_bytes=hx(r.edge_pair_min_volume_bytes))
        if solve:
            case["ilp"] = {}
            for mode in ("topology", "volume"):
                s = B.reference_solve(f, t, mode_volume=(mode == "volume"), threads=threads)
                case["ilp"][mode] = dict(strategy_per_op=s["strategy_per_op"], objective=hx([s["objective"]])[0],
                                         feasible=s["feasible"], optimal=s["optimal"])
    return case


def graph_json(g):
    return dict(operators=[dict(id=o.id, kind=o.kind,
                                inputs=[dict(name=t.name, shape=list(t.shape), element_size=t.element_size) for t in o.inputs],
                                outputs=[dict(name=t.name, shape=list(t.shape), element_size=t.element_size) for t in o.outputs],
                                axes=[dict(name=a.name, slices=[dict(tensor=s.tensor, dim=s.dim) for s in a.slices]) for a in o.axes])
                           for o in g.operators],
                edges=[dict(from_=e.from_, to=e.to, tensor=e.tensor) for e in g.edges])


def redist_case(shape, fd, fm, td, tm, local=8, intra=60e9, inter=6e9, nbytes=None):
    q = B.make_query(shape, fd, fm, td, tm, tensor_bytes=nbytes, local=local, intra=intra, inter=inter)
    r = B.reference_redistribute(q)
    d = dict(shape=list(shape), from_dims=list(fd), from_map=list(fm), to_dims=list(td), to_map=list(tm),
             local=local, intra=intra, inter=inter, tensor_bytes=q.tensor_bytes, status=int(r.status))
    if r.status == 0:
        dims, ushape, ufm, utm, ops, cts = r.plan()
        d.update(dims=list(dims), ushape=list(ushape), ufrom=list(ufm), uto=list(utm), ops=[list(o) for o in ops],
                 ct=list(cts), op_seconds=hx(r.op_seconds[:r.num_ops]), volume=hx([r.volume_bytes])[0],
                 seconds=hx([r.seconds])[0])
    return d


def main():
    out = {}
    # strategy tables (Table 3 and the config sizes)
    tabs = []
    for p in (1, 2, 3, 4):
        for N in (1, 2, 4, 8, 16, 32, 64, 128):
            deg, dm, md, dep = B.enumerate_with(B.reference().ref_enumerate, p, N)
            tabs.append(dict(p=p, N=N, degrees=deg.tolist(), device_map=dm.tolist(), matrix=md.tolist(),
                             depth=dep.tolist()))
    out["strategy_tables"] = tabs

    # redistribution goldens of the reference tests + random cases
    rc = [
        redist_case([8, 16], [2, 8], [1, 0], [8, 2], [1, 0]),            # Table 1, test_redistribution.cpp:43-51
        redist_case([8, 4], [4], [0, -1], [2, 2], [1, 0]),              # rank split, :64-76
        redist_case([4, 4, 4, 4, 4], [2, 2, 2, 2], [-1, 1, 2, -1, 3], [2, 2, 2, 2], [1, -1, -1, 0, 3]),  # Table 2
        redist_case([4, 4, 4, 4, 4], [4, 2, 2, 2], [-1, 1, 2, -1, 3], [4, 2, 2, 2], [1, -1, -1, 0, 3]),
        redist_case([4, 4], [2], [0, -1], [2], [-1, 0]),                 # single A2A, :148-160
        redist_case([8, 8], [2, 2], [0, 1], [2, 2], [1, 0]),             # swap -> fallback, :229-239
        redist_case([16, 16, 16, 16], [2, 2, 2, 2], [0, 1, 2, 3], [2, 2, 2, 2], [3, 2, 1, 0]),  # :369-377
        redist_case([8, 8], [2, 2], [0, 1], [2, 2], [1, -1], local=4),   # test_cost_model.cpp:296-306
        redist_case([6], [4], [0], [2, 2], [0]),                         # indivisible, :85-90
        redist_case([8, 8], [4], [0, -1], [2], [0, -1]),                 # incompatible totals, :78-82
        redist_case([12, 48], [4, 2], [1, 0], [2, 4], [0, 1], local=2),  # odd factor extents
    ]
    import random
    rng = random.Random(20260101)
    for i in range(300):
        dims, shape, fm, tm = fuzz.random_redist_case(rng)
        if i % 2:
            d2 = fuzz.random_matrix_with_total(rng, int(np.prod(dims)))
            tm = fuzz.random_map_for(rng, shape, d2)
        else:
            d2 = dims
        if i % 3 == 0:
            shape = [s * rng.choice([1, 3, 5]) for s in shape]
        rc.append(redist_case(shape, dims, fm, d2, tm, local=rng.choice([1, 2, 4, 8]), inter=rng.choice([6e9, 60e9])))
    out["redistributions"] = rc

    # builds: cfg1 (+ ILP), the aux-graph unit-test graphs, a join graph, memo aliasing
    from paper_2301_04285_b200.fuzz import elementwise_op
    from paper_2301_04285_b200.models import dense_op
    from paper_2301_04285_b200.graph import ClusterTopology, ComputationGraph, GraphEdge
    builds = [build_case("cfg1", *M.cfg1(), solve=True)]
    chain = ComputationGraph([dense_op("fc1", "matmul", "x0", 16, 16, 16, "x1"),
                              dense_op("fc2", "matmul", "x1", 16, 16, 16, "x2")], [GraphEdge("fc1", "fc2", "x1")])
    builds.append(build_case("chain_1x4", chain, ClusterTopology(1, 4, 60e9, 60e9, 32e9), solve=True))
    builds.append(build_case("chain_2x2", chain, ClusterTopology(2, 2, 60e9, 6e9, 32e9), solve=True))
    join = ComputationGraph([dense_op("a", "matmul", "x0", 16, 16, 16, "xa"), dense_op("b", "matmul", "x1", 16, 16, 16, "xb"),
                             elementwise_op("add", ["xa", "xb"], "sum", 16, 16)],
                            [GraphEdge("a", "add", "xa"), GraphEdge("b", "add", "xb")])
    builds.append(build_case("join_2x2", join, ClusterTopology(2, 2, 60e9, 6e9, 32e9), solve=True))
    # memo aliasing (SURVEY finding 3): same-shape tensors with element sizes 4 and 2
    alias = ComputationGraph(
        [dense_op("m1", "matmul", "x0", 64, 64, 64, "y1"), elementwise_op("e1", ["y1"], "z1", 64, 64),
         dense_op("m2", "matmul", "x2", 64, 64, 64, "y2"), elementwise_op("e2", ["y2"], "z2", 64, 64)],
        [GraphEdge("m1", "e1", "y1"), GraphEdge("m2", "e2", "y2")])
    for t in alias.operators[2].inputs + alias.operators[2].outputs + alias.operators[3].inputs + alias.operators[3].outputs:
        t.element_size = 2
    builds.append(build_case("memo_aliasing_2x4", alias, ClusterTopology(2, 4, 60e9, 6e9, 32e9)))
    builds.append(build_case("transformer_small_2x4",
                             M.build_transformer_layer(M.ModelConfig("transformer-layer", hidden=256, batch=4, seq=64)),
                             ClusterTopology(2, 4, 60e9, 6e9, 80e9), solve=True))
    builds.append(build_case("alexnet_2x8", M.build_alexnet_like(M.ModelConfig("alexnet-like", batch=64)),
                             ClusterTopology(2, 8, 60e9, 6e9, 256e9), solve=True))
    out["builds"] = builds
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "golden.json"), os.path.getsize(os.path.join(HERE, "golden.json")), "bytes")


if __name__ == "__main__":
    main()
