"""Seeded random inputs for parity tests (graphs and single redistributions).

`random_planning_instance` follows the shape of the reference's generator
(tests/test_support.hpp:350-409: short matmul/elementwise chains with residual
joins, <=16 devices); `random_graph` is a harsher generator for parity only
(odd extents, mixed element sizes, wider meshes, multi-consumer tensors)
whose graphs may make the reference throw — parity then means throwing the
same error class.
"""
from __future__ import annotations

import random
from typing import List, Tuple

from .graph import (AxisSlice, ClusterTopology, ComputationGraph, GraphEdge, OperatorAxis,
                    OperatorNode, TensorSpec, validate_graph)
from .models import dense_op


def elementwise_op(id, in_names, out_name, b, h, es=4):
    """tests/test_support.hpp:321-340."""
    d0 = OperatorAxis("d0", [AxisSlice(n, 0) for n in in_names] + [AxisSlice(out_name, 0)])
    d1 = OperatorAxis("d1", [AxisSlice(n, 1) for n in in_names] + [AxisSlice(out_name, 1)])
    return OperatorNode(id, "elementwise", [TensorSpec(n, [b, h], es) for n in in_names],
                        [TensorSpec(out_name, [b, h], es)], [d0, d1])


def _strategy_count(p, n_dev):
    import math
    n = n_dev.bit_length() - 1
    if n == 0:
        return 1
    return sum(math.factorial(i) * math.comb(p, i) * math.comb(n - 1, i - 1)
               for i in range(1, min(p, n) + 1))


def random_planning_instance(rng: random.Random, max_ops=5, search_cap=2e5):
    while True:
        g = ComputationGraph()
        ops = 2 + rng.randrange(max_ops - 1)
        b = 16 << rng.randrange(2)
        h = 16 << rng.randrange(3)
        widths = [h]
        for i in range(ops):
            in_name, out_name, id = f"t{i}", f"t{i + 1}", f"op{i}"
            if rng.randrange(2) == 0:
                nxt = 16 << rng.randrange(3)
                g.operators.append(dense_op(id, "matmul", in_name, b, widths[-1], nxt, out_name))
                widths.append(nxt)
            else:
                inputs = [in_name]
                for j in range(len(widths) - 2, 0, -1):
                    if widths[j] == widths[-1] and rng.randrange(3) == 0:
                        inputs.append(f"t{j}")
                        g.edges.append(GraphEdge(f"op{j - 1}", id, f"t{j}"))
                        break
                g.operators.append(elementwise_op(id, inputs, out_name, b, widths[-1]))
                widths.append(widths[-1])
            if i > 0:
                g.edges.append(GraphEdge(f"op{i - 1}", id, in_name))
        node_count = 1 << rng.randrange(3)
        local = 2 << rng.randrange(2)
        if node_count * local > 16:
            continue
        topo = ClusterTopology(node_count, local, 60e9, 60e9 if rng.randrange(4) == 0 else 6e9, 32e9)
        space = 1.0
        for op in g.operators:
            space *= _strategy_count(op.axis_count(), topo.total_devices())
        if space > search_cap:
            continue
        if not validate_graph(g).ok():
            continue
        return g, topo


def random_graph(rng: random.Random, max_ops=7, max_log2_devices=7, odd_extents=True,
                 mixed_element_sizes=False) -> Tuple[ComputationGraph, ClusterTopology]:
    """A DAG of dense / elementwise / 3-axis 'other' ops over rank-2 and
    rank-3 tensors. Extents are products of a power of two and an odd
    factor so many (not all) strategies divide."""
    def extent():
        e = 1 << rng.randrange(0, 8)
        if odd_extents and rng.randrange(3) == 0:
            e *= rng.choice([3, 5, 7, 9, 15])
        return e

    ops: List[OperatorNode] = []
    edges: List[GraphEdge] = []
    produced = []  # (op id, tensor spec)
    n_ops = 2 + rng.randrange(max_ops - 1)
    for i in range(n_ops):
        id = f"n{i}"
        kind = rng.randrange(3)
        es = rng.choice([1, 2, 4, 8]) if mixed_element_sizes else 4
        src = rng.choice(produced) if produced and rng.randrange(5) else None
        if kind == 0:  # dense
            if src and src[1].rank() == 2:
                rows, inn = src[1].shape
                in_name = src[1].name
                es = src[1].element_size
            else:
                rows, inn, in_name, src = extent(), extent(), f"x{i}", None
            op = dense_op(id, "matmul", in_name, rows, inn, extent(), f"y{i}")
            for t in op.inputs + op.outputs:
                t.element_size = es
        elif kind == 1:  # elementwise, 1-2 inputs
            if src and src[1].rank() == 2:
                shp, names, es = list(src[1].shape), [src[1].name], src[1].element_size
                # optional second input of the same shape
                cand = [p for p in produced if p[1].shape == shp and p[1].name != src[1].name]
                if cand and rng.randrange(2):
                    names.append(cand[0][1].name)
            else:
                shp, names, src = [extent(), extent()], [f"x{i}"], None
            op = elementwise_op(id, names, f"y{i}", shp[0], shp[1], es)
            if src:
                for nm in names[1:]:
                    pr = next(p for p in produced if p[1].name == nm)
                    edges.append(GraphEdge(pr[0], id, nm))
        else:  # rank-3 op with 3 axes
            if src and src[1].rank() == 3:
                shp, in_name, es = list(src[1].shape), src[1].name, src[1].element_size
            else:
                shp, in_name, src = [extent(), extent(), extent()], f"x{i}", None
            out = f"y{i}"
            op = OperatorNode(id, "other", [TensorSpec(in_name, shp, es)], [TensorSpec(out, shp, es)],
                              [OperatorAxis(f"a{d}", [AxisSlice(in_name, d), AxisSlice(out, d)])
                               for d in range(3)])
        if src:
            edges.append(GraphEdge(src[0], id, src[1].name))
        ops.append(op)
        for t in op.outputs:
            produced.append((id, t))
    nlog = rng.randrange(0, max_log2_devices + 1)
    local_log = rng.randrange(0, nlog + 1)
    topo = ClusterTopology(1 << (nlog - local_log), 1 << local_log, 60e9,
                           rng.choice([60e9, 6e9, 1.5e9, 25e9]), 32e9)
    return ComputationGraph(ops, edges), topo


def random_redist_case(rng: random.Random, max_elements=4096):
    """tests/test_support.hpp:275-319: a matrix, a shape and two maps over it."""
    depth = rng.randint(1, 3)
    dims = [4 if rng.randint(0, 1) else 2 for _ in range(depth)]
    rank = rng.randint(2, 4)
    while True:
        shape = [1 << rng.randrange(5) for _ in range(rank)]
        n = 1
        for s in shape:
            n *= s
        if n <= max_elements:
            break

    def ext(k):
        return dims[depth - 1 - k]

    def rmap():
        m = [-1] * rank
        ks = list(range(depth))
        rng.shuffle(ks)
        for k in ks:
            axes = list(range(rank))
            rng.shuffle(axes)
            if rng.randrange(4) == 0:
                continue
            for a in axes:
                if m[a] == -1 and shape[a] % ext(k) == 0 and shape[a] >= ext(k):
                    m[a] = k
                    break
        return m

    return dims, shape, rmap(), rmap()


def random_matrix_with_total(rng: random.Random, total: int):
    """tests/test_support.hpp:236-247."""
    dims = []
    rem = total
    while rem > 1:
        d = 4 if (rem % 4 == 0 and rng.randrange(2)) else 2
        dims.append(d)
        rem //= d
    rng.shuffle(dims)
    return dims


def random_map_for(rng: random.Random, shape, dims):
    """tests/test_support.hpp:250-273."""
    depth = len(dims)
    rank = len(shape)
    m = [-1] * rank
    ks = list(range(depth))
    rng.shuffle(ks)
    for k in ks:
        if rng.randrange(4) == 0:
            continue
        axes = list(range(rank))
        rng.shuffle(axes)
        e = dims[depth - 1 - k]
        for a in axes:
            if m[a] == -1 and shape[a] % e == 0 and shape[a] >= e:
                m[a] = k
                break
    return m
