"""ctypes bindings of the two CPU checkers — TEST INFRASTRUCTURE ONLY.

  oracle()     -> oracle/liboracle.so           (C restatement, taps_oracle.c)
  reference()  -> oracle/_ref/libtopoplan_ref.so (the reference itself, ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from paper_2301_04285_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtopoplan_ref.so")

P = C.POINTER
_oracle = None
_ref = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        lib = C.CDLL(ORACLE_SO)
        for fn in ("oracle_build", "oracle_build_unmemoized"):
            getattr(lib, fn).argtypes = [P(abi.tp_graph_desc), P(abi.tp_topology_desc),
                                         P(abi.tp_aux_index), P(abi.tp_cost_tensors), P(C.c_int32)]
            getattr(lib, fn).restype = C.c_int
        lib.oracle_sizes.argtypes = [P(abi.tp_graph_desc), P(abi.tp_topology_desc), P(C.c_int64),
                                     P(C.c_int64), P(C.c_int64)]
        lib.oracle_sizes.restype = C.c_int
        lib.oracle_redistribute.argtypes = [P(abi.tp_redist_query), P(abi.tp_redist_result)]
        lib.oracle_redistribute.restype = C.c_int
        lib.oracle_enumerate.argtypes = [C.c_int32, C.c_int64, P(C.c_int64), P(C.c_int32),
                                         P(C.c_int64), P(C.c_int32)]
        lib.oracle_enumerate.restype = C.c_int64
        lib.oracle_strategy_count.argtypes = [C.c_int32, C.c_int64]
        lib.oracle_strategy_count.restype = C.c_int64
        lib.oracle_ct_allreduce.argtypes = [C.c_int32, P(C.c_int64), C.c_int32, P(C.c_int32), C.c_int64]
        lib.oracle_ct_allreduce.restype = C.c_int64
        lib.oracle_ct_allgather_dim.argtypes = [C.c_int32, P(C.c_int64), C.c_int32, P(C.c_int32),
                                                C.c_int32, C.c_int64, P(C.c_int64), P(C.c_int64),
                                                P(C.c_int64)]
        lib.oracle_ct_allgather_dim.restype = None
        _oracle = lib
    return _oracle


def have_reference() -> bool:
    return os.path.exists(REF_SO)


def reference() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        lib.ref_build.argtypes = [P(abi.tp_graph_desc), P(abi.tp_topology_desc), P(abi.tp_aux_index),
                                  P(abi.tp_cost_tensors)]
        lib.ref_build.restype = C.c_int
        lib.ref_build_unmemoized.argtypes = [P(abi.tp_graph_desc), P(abi.tp_topology_desc),
                                             P(abi.tp_cost_tensors)]
        lib.ref_build_unmemoized.restype = C.c_int
        lib.ref_bench_build.argtypes = [P(abi.tp_graph_desc), P(abi.tp_topology_desc), C.c_int,
                                        C.c_int, P(C.c_double), P(C.c_int64)]
        lib.ref_bench_build.restype = C.c_int
        lib.ref_redistribute.argtypes = [P(abi.tp_redist_query), P(abi.tp_redist_result)]
        lib.ref_redistribute.restype = C.c_int
        lib.ref_enumerate.argtypes = [C.c_int32, C.c_int64, P(C.c_int64), P(C.c_int32), P(C.c_int64),
                                      P(C.c_int32)]
        lib.ref_enumerate.restype = C.c_int64
        lib.ref_strategy_count.argtypes = [C.c_int32, C.c_int64]
        lib.ref_strategy_count.restype = C.c_int64
        lib.ref_ct_allreduce.argtypes = [C.c_int32, P(C.c_int64), C.c_int32, P(C.c_int32), C.c_int64]
        lib.ref_ct_allreduce.restype = C.c_int64
        lib.ref_ct_allgather_dim.argtypes = [C.c_int32, P(C.c_int64), C.c_int32, P(C.c_int32),
                                             C.c_int32, C.c_int64, P(C.c_int64), P(C.c_int64),
                                             P(C.c_int64)]
        lib.ref_ct_allgather_dim.restype = None
        lib.ref_solve.argtypes = [P(abi.tp_graph_desc), P(abi.tp_topology_desc), C.c_int, C.c_double,
                                  C.c_int, C.c_int64, P(abi.tp_cost_tensors), P(C.c_int32),
                                  P(C.c_double), P(C.c_int32), P(C.c_int32), P(C.c_double),
                                  P(C.c_int64)]
        lib.ref_solve.restype = C.c_int
        lib.ref_price_assignments.argtypes = [P(abi.tp_graph_desc), P(abi.tp_topology_desc), P(C.c_int32),
                                              C.c_int, P(C.c_double), P(C.c_double), P(C.c_double)]
        lib.ref_price_assignments.restype = C.c_int
        lib.ref_export_lp.argtypes = [P(abi.tp_graph_desc), P(abi.tp_topology_desc), C.c_int,
                                      C.c_double, C.c_char_p, C.c_int64]
        lib.ref_export_lp.restype = C.c_int64
        lib.ref_composer_json.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_char_p,
                                          C.c_int64]
        lib.ref_composer_json.restype = C.c_int64
        lib.ref_model_json.argtypes = [C.c_char_p, C.c_char_p, C.c_int64]
        lib.ref_model_json.restype = C.c_int64
        lib.ref_last_error.argtypes = []
        lib.ref_last_error.restype = C.c_char_p
        _ref = lib
    return _ref


@dataclass
class BuildResult:
    status: int
    kind: int = 0
    node_base: Optional[np.ndarray] = None
    edge_base: Optional[np.ndarray] = None
    edge_from_op: Optional[np.ndarray] = None
    edge_to_op: Optional[np.ndarray] = None
    in_degree: Optional[np.ndarray] = None
    out_degree: Optional[np.ndarray] = None
    topo_order: Optional[np.ndarray] = None
    node_intra_cost_s: Optional[np.ndarray] = None
    node_intra_volume_bytes: Optional[np.ndarray] = None
    node_memory_bytes: Optional[np.ndarray] = None
    edge_cost_s: Optional[np.ndarray] = None
    edge_volume_bytes: Optional[np.ndarray] = None
    edge_memory_bytes: Optional[np.ndarray] = None
    records: Optional[np.ndarray] = None
    row_min_cost_s: Optional[np.ndarray] = None
    row_min_volume_bytes: Optional[np.ndarray] = None
    edge_pair_min_cost_s: Optional[np.ndarray] = None
    edge_pair_min_volume_bytes: Optional[np.ndarray] = None
    extra: dict = field(default_factory=dict)


def alloc_outputs(num_ops, num_edges, num_nodes, num_aux_edges, num_rows, records=True):
    r = BuildResult(status=-1)
    r.node_base = np.zeros(num_ops + 1, np.int64)
    r.edge_base = np.zeros(num_edges + 1, np.int64)
    r.edge_from_op = np.zeros(max(num_edges, 1), np.int32)
    r.edge_to_op = np.zeros(max(num_edges, 1), np.int32)
    r.in_degree = np.zeros(max(num_ops, 1), np.int32)
    r.out_degree = np.zeros(max(num_ops, 1), np.int32)
    r.topo_order = np.zeros(max(num_ops, 1), np.int32)
    r.node_intra_cost_s = np.zeros(max(num_nodes, 1))
    r.node_intra_volume_bytes = np.zeros(max(num_nodes, 1))
    r.node_memory_bytes = np.zeros(max(num_nodes, 1))
    r.edge_cost_s = np.zeros(max(num_aux_edges, 1))
    r.edge_volume_bytes = np.zeros(max(num_aux_edges, 1))
    r.edge_memory_bytes = np.zeros(max(num_aux_edges, 1))
    r.records = np.zeros(max(num_aux_edges, 1) * 40, np.uint8) if records else None
    r.row_min_cost_s = np.zeros(max(num_rows, 1))
    r.row_min_volume_bytes = np.zeros(max(num_rows, 1))
    r.edge_pair_min_cost_s = np.zeros(max(num_edges, 1))
    r.edge_pair_min_volume_bytes = np.zeros(max(num_edges, 1))
    return r


def index_struct(r: BuildResult) -> abi.tp_aux_index:
    return abi.tp_aux_index(abi.ptr(r.node_base, C.c_int64), abi.ptr(r.edge_base, C.c_int64),
                            abi.ptr(r.edge_from_op, C.c_int32), abi.ptr(r.edge_to_op, C.c_int32),
                            abi.ptr(r.in_degree, C.c_int32), abi.ptr(r.out_degree, C.c_int32),
                            abi.ptr(r.topo_order, C.c_int32))


def cost_struct(r: BuildResult) -> abi.tp_cost_tensors:
    f = lambda a: abi.ptr(a, C.c_double) if a is not None else None
    return abi.tp_cost_tensors(f(r.node_intra_cost_s), f(r.node_intra_volume_bytes),
                               f(r.node_memory_bytes), f(r.edge_cost_s), f(r.edge_volume_bytes),
                               f(r.edge_memory_bytes),
                               r.records.ctypes.data_as(C.c_void_p) if r.records is not None else None,
                               f(r.row_min_cost_s), f(r.row_min_volume_bytes),
                               f(r.edge_pair_min_cost_s), f(r.edge_pair_min_volume_bytes))


def sizes(flat, topo):
    d, t = flat.desc(), topo.desc()
    nn, ne, nr = C.c_int64(), C.c_int64(), C.c_int64()
    st = oracle().oracle_sizes(C.byref(d), C.byref(t), C.byref(nn), C.byref(ne), C.byref(nr))
    if st != 0:
        return None
    return nn.value, ne.value, nr.value


def _trim(r: BuildResult, nn, ne, nr, num_ops, num_edges):
    r.node_intra_cost_s = r.node_intra_cost_s[:nn]
    r.node_intra_volume_bytes = r.node_intra_volume_bytes[:nn]
    r.node_memory_bytes = r.node_memory_bytes[:nn]
    r.edge_cost_s = r.edge_cost_s[:ne]
    r.edge_volume_bytes = r.edge_volume_bytes[:ne]
    r.edge_memory_bytes = r.edge_memory_bytes[:ne]
    if r.records is not None:
        r.records = r.records[: ne * 40]
    r.row_min_cost_s = r.row_min_cost_s[:nr]
    r.row_min_volume_bytes = r.row_min_volume_bytes[:nr]
    if r.edge_pair_min_cost_s is not None:
        r.edge_pair_min_cost_s = r.edge_pair_min_cost_s[:num_edges]
        r.edge_pair_min_volume_bytes = r.edge_pair_min_volume_bytes[:num_edges]
    r.edge_from_op = r.edge_from_op[:num_edges]
    r.edge_to_op = r.edge_to_op[:num_edges]
    r.in_degree = r.in_degree[:num_ops]
    r.out_degree = r.out_degree[:num_ops]
    r.topo_order = r.topo_order[:num_ops]
    return r


def oracle_build(flat, topo, memoize=True, records=True) -> BuildResult:
    s = sizes(flat, topo)
    nn, ne, nr = s if s else (0, 0, 0)
    r = alloc_outputs(flat.num_ops, flat.num_edges, nn, ne, nr, records)
    d, t = flat.desc(), topo.desc()
    idx, out = index_struct(r), cost_struct(r)
    kind = C.c_int32()
    fn = oracle().oracle_build if memoize else oracle().oracle_build_unmemoized
    r.status = fn(C.byref(d), C.byref(t), C.byref(idx), C.byref(out), C.byref(kind))
    r.kind = kind.value
    return _trim(r, nn, ne, nr, flat.num_ops, flat.num_edges)


def reference_build(flat, topo, records=True) -> BuildResult:
    s = sizes(flat, topo)
    nn, ne, nr = s if s else (0, 0, 0)
    r = alloc_outputs(flat.num_ops, flat.num_edges, nn, ne, nr, records)
    d, t = flat.desc(), topo.desc()
    idx, out = index_struct(r), cost_struct(r)
    r.status = reference().ref_build(C.byref(d), C.byref(t), C.byref(idx), C.byref(out))
    r.extra["message"] = reference().ref_last_error().decode()
    return _trim(r, nn, ne, nr, flat.num_ops, flat.num_edges)


def reference_build_unmemoized(flat, topo) -> BuildResult:
    s = sizes(flat, topo)
    nn, ne, nr = s
    r = alloc_outputs(flat.num_ops, flat.num_edges, nn, ne, nr, False)
    d, t = flat.desc(), topo.desc()
    out = cost_struct(r)
    r.status = reference().ref_build_unmemoized(C.byref(d), C.byref(t), C.byref(out))
    return _trim(r, nn, ne, nr, flat.num_ops, flat.num_edges)


def make_query(shape, from_dims, from_map, to_dims, to_map, tensor_bytes=None, local=8,
               intra=60e9, inter=6e9):
    """A tp_redist_query plus the numpy buffers it points into."""
    shape = np.asarray(shape, np.int64)
    fd = np.asarray(list(from_dims) or [0], np.int64)
    td = np.asarray(list(to_dims) or [0], np.int64)
    fm = np.asarray(from_map, np.int32)
    tm = np.asarray(to_map, np.int32)
    if tensor_bytes is None:
        tensor_bytes = 4.0 * float(np.prod(shape))
    q = abi.tp_redist_query(len(shape), abi.ptr(shape, C.c_int64), len(from_dims),
                            abi.ptr(fd, C.c_int64), abi.ptr(fm, C.c_int32), len(to_dims),
                            abi.ptr(td, C.c_int64), abi.ptr(tm, C.c_int32), tensor_bytes, local,
                            intra, inter)
    q._keep = (shape, fd, td, fm, tm)
    return q


def oracle_redistribute(q) -> abi.tp_redist_result:
    r = abi.tp_redist_result()
    oracle().oracle_redistribute(C.byref(q), C.byref(r))
    return r


def reference_redistribute(q) -> abi.tp_redist_result:
    r = abi.tp_redist_result()
    st = reference().ref_redistribute(C.byref(q), C.byref(r))
    if st != 0:
        r.status = -st
    return r


def enumerate_with(lib_fn, p, N):
    n = lib_fn(p, N, None, None, None, None)
    if n < 0:
        return None
    deg = np.zeros(max(n * p, 1), np.int64)
    dm = np.zeros(max(n * p, 1), np.int32)
    md = np.zeros(max(n * p, 1), np.int64)
    dep = np.zeros(max(n, 1), np.int32)
    lib_fn(p, N, abi.ptr(deg, C.c_int64), abi.ptr(dm, C.c_int32), abi.ptr(md, C.c_int64),
           abi.ptr(dep, C.c_int32))
    return (deg[: n * p].reshape(n, p), dm[: n * p].reshape(n, p), md[: n * p].reshape(n, p),
            dep[:n])


def reference_solve(flat, topo, mode_volume=False, memory_bound=None, threads=1,
                    max_nodes=200_000_000, given: Optional[BuildResult] = None):
    d, t = flat.desc(), topo.desc()
    if memory_bound is None:
        memory_bound = topo.device_memory
    per_op = np.zeros(max(flat.num_ops, 1), np.int32)
    obj, feas, opt, root, nodes = C.c_double(), C.c_int32(), C.c_int32(), C.c_double(), C.c_int64()
    g = cost_struct(given) if given is not None else None
    st = reference().ref_solve(C.byref(d), C.byref(t), int(mode_volume), memory_bound, threads,
                               max_nodes, C.byref(g) if g is not None else None,
                               abi.ptr(per_op, C.c_int32), C.byref(obj), C.byref(feas),
                               C.byref(opt), C.byref(root), C.byref(nodes))
    if st != 0:
        raise RuntimeError(reference().ref_last_error().decode())
    return dict(strategy_per_op=per_op[: flat.num_ops].tolist(), objective=obj.value,
                feasible=bool(feas.value), optimal=bool(opt.value), root_bound=root.value,
                nodes=nodes.value)


def reference_price_assignments(flat, topo, asg):
    """The reference's price_assignment (aux_graph.hpp:326-348) of every row
    of asg [k, num_ops] on its own build: (topology cost, volume cost,
    memory) arrays of length k."""
    asg = np.ascontiguousarray(asg, dtype=np.int32)
    k = asg.shape[0]
    d, t = flat.desc(), topo.desc()
    c, v, m = (np.zeros(max(k, 1)) for _ in range(3))
    st = reference().ref_price_assignments(C.byref(d), C.byref(t), abi.ptr(asg, C.c_int32), k,
                                           abi.ptr(c, C.c_double), abi.ptr(v, C.c_double),
                                           abi.ptr(m, C.c_double))
    if st != 0:
        raise RuntimeError(reference().ref_last_error().decode())
    return c[:k], v[:k], m[:k]


def reference_export_lp(flat, topo, mode_volume=False, memory_bound=None) -> bytes:
    """export_lp(formulate(...)) (solver.hpp:578-600) of the reference's own
    build, as bytes."""
    d, t = flat.desc(), topo.desc()
    mem = topo.device_memory if memory_bound is None else memory_bound
    n = reference().ref_export_lp(C.byref(d), C.byref(t), int(mode_volume), mem, None, 0)
    if n < 0:
        raise RuntimeError(reference().ref_last_error().decode())
    buf = C.create_string_buffer(n + 1)
    reference().ref_export_lp(C.byref(d), C.byref(t), int(mode_volume), mem, buf, n + 1)
    return buf.raw[:n]


def reference_bench(flat, topo, iters=1, threads=1):
    d, t = flat.desc(), topo.desc()
    secs, edges = C.c_double(), C.c_int64()
    st = reference().ref_bench_build(C.byref(d), C.byref(t), iters, threads, C.byref(secs),
                                     C.byref(edges))
    if st != 0:
        raise RuntimeError(reference().ref_last_error().decode())
    return secs.value, edges.value


def reference_bench_sweep(pairs, threads=1):
    """(seconds, aux edges) of building every (flat, topo) scenario with the
    reference on a pool of `threads` host threads."""
    n = len(pairs)
    ds = [f.desc() for f, _ in pairs]
    ts = [t.desc() for _, t in pairs]
    gp = (C.POINTER(abi.tp_graph_desc) * max(n, 1))(*[C.pointer(d) for d in ds])
    tp = (C.POINTER(abi.tp_topology_desc) * max(n, 1))(*[C.pointer(d) for d in ts])
    secs, edges = C.c_double(), C.c_int64()
    st = reference().ref_bench_sweep(gp, tp, n, threads, C.byref(secs), C.byref(edges))
    if st != 0:
        raise RuntimeError(reference().ref_last_error().decode())
    return secs.value, edges.value
