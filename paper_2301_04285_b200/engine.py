"""Python face of the CUDA cost-tensor engine (include/taps_b200.h).

`build_cost_tensors(graph, topo)` is the drop-in for the reference's
`topoplan::build_auxiliary_graph(graph, topo, mode)`
(/root/reference/proj/include/topoplan/aux_graph.hpp:211-315): it returns
the same quantities (aux node/edge payloads in the reference's index order)
as numpy arrays. `Plan` is the split API for device-resident, repeated or
sharded builds (torch tensors as device memory; torch is plumbing only).
There is no CPU path: without the CUDA library or a GPU every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Tuple, Union

import numpy as np

from . import abi
from .graph import ClusterTopology, ComputationGraph, FlatGraph, flatten


def _check(lib, status):
    if status != abi.TP_OK:
        abi.raise_for_status(status, lib.tp_last_error().decode(), lib.tp_last_error_kind())


def _flat(graph) -> FlatGraph:
    return graph if isinstance(graph, FlatGraph) else flatten(graph)


@dataclass
class CostTensors:
    """Cost tensors of one build, reference index order (aux_graph.hpp:93-98)."""
    node_base: np.ndarray
    edge_base: np.ndarray
    edge_from_op: np.ndarray
    edge_to_op: np.ndarray
    in_degree: np.ndarray
    out_degree: np.ndarray
    topo_order: np.ndarray
    node_intra_cost_s: np.ndarray
    node_intra_volume_bytes: np.ndarray
    node_memory_bytes: np.ndarray
    edge_cost_s: np.ndarray
    edge_volume_bytes: np.ndarray
    edge_memory_bytes: np.ndarray
    records: Optional[np.ndarray] = None
    row_min_cost_s: Optional[np.ndarray] = None
    row_min_volume_bytes: Optional[np.ndarray] = None
    edge_pair_min_cost_s: Optional[np.ndarray] = None  # solver.hpp:254-255 pair_min
    edge_pair_min_volume_bytes: Optional[np.ndarray] = None
    sizes: dict = field(default_factory=dict)

    def strategies_of(self, op: int) -> int:
        return int(self.node_base[op + 1] - self.node_base[op])

    def edge_id(self, e: int, su: int, sw: int) -> int:
        """AuxiliaryGraph::edge_id (aux_graph.hpp:93-98)."""
        return int(self.edge_base[e] + su * self.strategies_of(int(self.edge_to_op[e])) + sw)

    def virtual_edges(self):
        """(op, aux node) of every virtual source edge (aux_graph.hpp:298-312);
        their payload is the node's own (intra cost, intra volume, memory)."""
        out = []
        for op in range(len(self.node_base) - 1):
            if self.in_degree[op] == 0:
                out.extend((op, n) for n in range(int(self.node_base[op]), int(self.node_base[op + 1])))
        return out

    def price_assignment(self, assignment, mode: str = "topology") -> Tuple[float, float]:
        """price_assignment (aux_graph.hpp:326-348): topological order, a
        source's virtual edge first, then its in-edges ascending."""
        cost = 0.0
        mem = 0.0
        n_edges = len(self.edge_to_op)
        in_edges = [[] for _ in range(len(self.node_base) - 1)]
        for e in range(n_edges):
            in_edges[int(self.edge_to_op[e])].append(e)
        for op in self.topo_order:
            op = int(op)
            node = int(self.node_base[op]) + int(assignment[op])
            if self.in_degree[op] == 0:
                cost += float(self.node_intra_volume_bytes[node] if mode == "volume"
                              else self.node_intra_cost_s[node])
                mem += float(self.node_memory_bytes[node])
            for e in in_edges[op]:
                u = int(self.edge_from_op[e])
                a = self.edge_id(e, int(assignment[u]), int(assignment[op]))
                cost += float(self.edge_volume_bytes[a] if mode == "volume" else self.edge_cost_s[a])
                mem += float(self.edge_memory_bytes[a])
        return cost, mem


class Plan:
    """tp_plan: host analysis once, device execution many times."""

    def __init__(self, graph: Union[ComputationGraph, FlatGraph], topo: ClusterTopology, device: int = -1):
        self.lib = abi.load_engine()
        self.flat = _flat(graph)
        self.topo = topo
        self._desc = self.flat.desc()
        self._tdesc = topo.desc()
        h = C.c_void_p()
        _check(self.lib, self.lib.tp_plan_create(C.byref(self._desc), C.byref(self._tdesc), device, C.byref(h)))
        self.handle = h
        s = abi.tp_plan_sizes_t()
        _check(self.lib, self.lib.tp_plan_sizes(self.handle, C.byref(s)))
        self.sizes = {k: getattr(s, k) for k, _ in abi.tp_plan_sizes_t._fields_}

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            self.lib.tp_plan_destroy(h)
            self.handle = None

    def index(self) -> dict:
        n_ops, n_e = self.flat.num_ops, self.flat.num_edges
        ix = dict(node_base=np.zeros(n_ops + 1, np.int64), edge_base=np.zeros(n_e + 1, np.int64),
                  edge_from_op=np.zeros(max(n_e, 1), np.int32), edge_to_op=np.zeros(max(n_e, 1), np.int32),
                  in_degree=np.zeros(max(n_ops, 1), np.int32), out_degree=np.zeros(max(n_ops, 1), np.int32),
                  topo_order=np.zeros(max(n_ops, 1), np.int32))
        st = abi.tp_aux_index(*(abi.ptr(ix[k], C.c_int64 if ix[k].dtype == np.int64 else C.c_int32)
                                for k, _ in abi.tp_aux_index._fields_))
        _check(self.lib, self.lib.tp_plan_index(self.handle, C.byref(st)))
        for k, n in (("edge_from_op", n_e), ("edge_to_op", n_e), ("in_degree", n_ops),
                     ("out_degree", n_ops), ("topo_order", n_ops)):
            ix[k] = ix[k][:n]
        return ix

    def upload(self, stream: int = 0):
        _check(self.lib, self.lib.tp_plan_upload(self.handle, C.c_void_p(stream or None)))

    def execute(self, out: abi.tp_cost_tensors, edge_range=(0, -1), skip_nodes=False, stream: int = 0):
        """Asynchronous on `stream` into DEVICE pointers."""
        o = abi.tp_build_opts(edge_range[0], edge_range[1], int(skip_nodes), -1, C.c_void_p(stream or None))
        _check(self.lib, self.lib.tp_plan_execute(self.handle, C.byref(o), C.byref(out)))

    def check_errors(self):
        _check(self.lib, self.lib.tp_plan_check_errors(self.handle))

    def set_profile_events(self, start, stop):
        """torch.cuda.Event pair recorded around the fan-out kernel (K4)."""
        _check(self.lib, self.lib.tp_plan_set_profile_events(
            self.handle, C.c_void_p(start.cuda_event if start is not None else None),
            C.c_void_p(stop.cuda_event if stop is not None else None)))

    def set_timeline(self, on: bool = True):
        """Record device timestamps of the build phases (diagnostics)."""
        _check(self.lib, self.lib.tp_plan_set_timeline(self.handle, int(on)))

    def timeline(self) -> dict:
        """ns after kernel start of the last execute (synchronises): node rows
        done, first pair done, pairs done, first fan-out tile, kernel end."""
        v = (C.c_int64 * 5)()
        _check(self.lib, self.lib.tp_plan_timeline(self.handle, v))
        return dict(zip(("rows", "first_pair", "pairs", "first_fanout", "end"), list(v)))

    def timeline_detail(self):
        """Per-item traces of the last execute (ns): pairs as [start, duration,
        edge class], node rows as [start, duration], fan-out ranges as
        [start, wait, duration]."""
        import numpy as np
        res = []
        for sec, w in ((0, 3), (1, 2), (2, 3), (3, 8), (4, 1)):
            n = C.c_int64(0)
            _check(self.lib, self.lib.tp_plan_timeline_detail(self.handle, sec, None, C.byref(n)))
            v = np.zeros((n.value, w), np.uint32)
            _check(self.lib, self.lib.tp_plan_timeline_detail(
                self.handle, sec, v.ctypes.data_as(C.POINTER(C.c_uint32)), C.byref(n)))
            res.append(v)
        return tuple(res)

    def set_pair_form(self, form: int):
        """0 = by size (default), 1 = warp per class pair, 2 = thread per pair."""
        _check(self.lib, self.lib.tp_plan_set_pair_form(self.handle, form))

    def last_launches(self) -> int:
        return int(self.lib.tp_plan_last_launches(self.handle))

    def set_bandwidth(self, intra_bandwidth: float, inter_bandwidth: float):
        """Re-price under other intra/inter bandwidths without re-analysing
        (tp_plan_set_bandwidth); the next execute rebuilds."""
        _check(self.lib, self.lib.tp_plan_set_bandwidth(self.handle, float(intra_bandwidth), float(inter_bandwidth)))
        t = self.topo
        self.topo = ClusterTopology(t.node_count, t.local_device_num, float(intra_bandwidth), float(inter_bandwidth),
                                    t.device_memory)

    def price_assignments(self, tensors: dict, assignments, stream: int = 0):
        """price_assignment (aux_graph.hpp:326-348) of every row of
        `assignments` (a CUDA int32 tensor [k, num_ops]) against this plan's
        device cost tensors (dict of the six tensors, as executed): returns
        CUDA float64 tensors (topology-mode cost, volume-mode cost, memory)."""
        import torch
        a = assignments.to(torch.int32).contiguous()
        k = int(a.shape[0]) if a.dim() == 2 else 0
        outs = [torch.empty(max(k, 1), dtype=torch.float64, device=a.device) for _ in range(3)]
        ptr = lambda x: C.cast(C.c_void_p(x.data_ptr()), C.POINTER(C.c_double))
        ts = device_cost_struct(tensors)
        _check(self.lib, self.lib.tp_plan_price_assignments(
            self.handle, C.byref(ts), C.cast(C.c_void_p(a.data_ptr()), C.POINTER(C.c_int32)), k,
            ptr(outs[0]), ptr(outs[1]), ptr(outs[2]), C.c_void_p(stream or None)))
        return tuple(o[:k] for o in outs)

    def execute_host(self, records=False, row_min=False, edge_range=(0, -1), skip_nodes=False,
                     pinned=False, scratch=False) -> CostTensors:
        """Synchronous build into HOST buffers (pinned if requested); with
        `scratch` on the calling thread's reused device memory
        (tp_plan_execute_host_scratch) when the plan has none of its own."""
        ix = self.index()
        e0, e1 = edge_range
        if e1 < 0:
            e1 = self.flat.num_edges
        eb = ix["edge_base"]
        ne = int(eb[e1] - eb[e0])
        nn = self.sizes["num_aux_nodes"]
        rows = _row_counts(ix, e0, e1)
        alloc = _pinned_empty if pinned else (lambda n, dt: np.zeros(n, dt))
        ct = CostTensors(
            node_intra_cost_s=alloc(max(nn, 1), np.float64), node_intra_volume_bytes=alloc(max(nn, 1), np.float64),
            node_memory_bytes=alloc(max(nn, 1), np.float64), edge_cost_s=alloc(max(ne, 1), np.float64),
            edge_volume_bytes=alloc(max(ne, 1), np.float64), edge_memory_bytes=alloc(max(ne, 1), np.float64),
            records=alloc(max(ne, 1) * 40, np.uint8) if records else None,
            row_min_cost_s=alloc(max(rows, 1), np.float64) if row_min else None,
            row_min_volume_bytes=alloc(max(rows, 1), np.float64) if row_min else None,
            edge_pair_min_cost_s=alloc(max(e1 - e0, 1), np.float64) if row_min else None,
            edge_pair_min_volume_bytes=alloc(max(e1 - e0, 1), np.float64) if row_min else None,
            sizes=dict(self.sizes), **ix)
        out = cost_struct(ct)
        o = abi.tp_build_opts(e0, e1, int(skip_nodes), -1, None)
        fn = self.lib.tp_plan_execute_host_scratch if scratch else self.lib.tp_plan_execute_host
        _check(self.lib, fn(self.handle, C.byref(o), None, C.byref(out)))
        _trim(ct, nn, ne, rows, e1 - e0)
        return ct


def _multi(self, devices, records=False, row_min=False, pinned=False) -> CostTensors:
    """tp_plan_execute_host_multi: the graph's edges in contiguous ranges
    balanced by aux edges, range i built on devices[i] and its slice copied
    straight into the host arrays at its offset."""
    ix = self.index()
    ne, nn = self.sizes["num_aux_edges"], self.sizes["num_aux_nodes"]
    n_e = self.flat.num_edges
    rows = _row_counts(ix, 0, n_e)
    alloc = _pinned_empty if pinned else (lambda n, dt: np.zeros(n, dt))
    ct = CostTensors(
        node_intra_cost_s=alloc(max(nn, 1), np.float64), node_intra_volume_bytes=alloc(max(nn, 1), np.float64),
        node_memory_bytes=alloc(max(nn, 1), np.float64), edge_cost_s=alloc(max(ne, 1), np.float64),
        edge_volume_bytes=alloc(max(ne, 1), np.float64), edge_memory_bytes=alloc(max(ne, 1), np.float64),
        records=alloc(max(ne, 1) * 40, np.uint8) if records else None,
        row_min_cost_s=alloc(max(rows, 1), np.float64) if row_min else None,
        row_min_volume_bytes=alloc(max(rows, 1), np.float64) if row_min else None,
        edge_pair_min_cost_s=alloc(max(n_e, 1), np.float64) if row_min else None,
        edge_pair_min_volume_bytes=alloc(max(n_e, 1), np.float64) if row_min else None,
        sizes=dict(self.sizes), **ix)
    out = cost_struct(ct)
    devs = np.ascontiguousarray(devices, dtype=np.int32)
    self._multi_keep = (ct, out, devs)
    _check(self.lib, self.lib.tp_plan_execute_host_multi(self.handle, abi.ptr(devs, C.c_int32), len(devs), None,
                                                         C.byref(out)))
    _trim(ct, nn, ne, rows, n_e)
    return ct


Plan.execute_host_multi = _multi


def _export_lp(self, ct: CostTensors, path: str, mode: str = "topology", device_memory=None) -> int:
    """topoplan::export_lp(formulate(aux, mode, device_memory)) of this build
    (ct = execute_host's result) written to `path` (tp_plan_export_lp);
    returns the bytes written."""
    out = cost_struct(ct)
    n = C.c_int64()
    mem = self.topo.device_memory if device_memory is None else device_memory
    _check(self.lib, self.lib.tp_plan_export_lp(self.handle, C.byref(out), int(mode == "volume"), float(mem),
                                                os.fsencode(path), C.byref(n)))
    return n.value


Plan.export_lp = _export_lp


def build_cost_tensors_multi(graph, topo: ClusterTopology, devices, records=False, row_min=False,
                             pinned=False) -> CostTensors:
    """The drop-in for build_auxiliary_graph on several GPUs of this process
    (tp_plan_execute_host_multi): bit-identical to build_cost_tensors."""
    plan = Plan(graph, topo, int(devices[0]))
    return plan.execute_host_multi(devices, records=records, row_min=row_min, pinned=pinned)


def _row_counts(ix, e0, e1):
    nb = ix["node_base"]
    return int(sum(int(nb[ix["edge_from_op"][e] + 1] - nb[ix["edge_from_op"][e]]) for e in range(e0, e1)))


def _pinned_empty(n, dtype):
    import torch
    tdt = {np.float64: torch.float64, np.uint8: torch.uint8}[dtype]
    return torch.empty(n, dtype=tdt, pin_memory=True).numpy()


def _trim(ct: CostTensors, nn, ne, rows, nedges):
    for k in ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes"):
        setattr(ct, k, getattr(ct, k)[:nn])
    for k in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes"):
        setattr(ct, k, getattr(ct, k)[:ne])
    if ct.records is not None:
        ct.records = ct.records[: ne * 40]
    if ct.row_min_cost_s is not None:
        ct.row_min_cost_s = ct.row_min_cost_s[:rows]
        ct.row_min_volume_bytes = ct.row_min_volume_bytes[:rows]
    if ct.edge_pair_min_cost_s is not None:
        ct.edge_pair_min_cost_s = ct.edge_pair_min_cost_s[:nedges]
        ct.edge_pair_min_volume_bytes = ct.edge_pair_min_volume_bytes[:nedges]


def cost_struct(ct) -> abi.tp_cost_tensors:
    f = lambda a: abi.ptr(a, C.c_double) if a is not None else None
    return abi.tp_cost_tensors(
        f(ct.node_intra_cost_s), f(ct.node_intra_volume_bytes), f(ct.node_memory_bytes),
        f(ct.edge_cost_s), f(ct.edge_volume_bytes), f(ct.edge_memory_bytes),
        ct.records.ctypes.data_as(C.c_void_p) if ct.records is not None else None,
        f(ct.row_min_cost_s), f(ct.row_min_volume_bytes),
        f(getattr(ct, "edge_pair_min_cost_s", None)), f(getattr(ct, "edge_pair_min_volume_bytes", None)))


def device_cost_struct(tensors: dict) -> abi.tp_cost_tensors:
    """tp_cost_tensors of torch CUDA tensors (missing keys -> NULL)."""
    def p(k, t=C.c_double):
        x = tensors.get(k)
        return C.cast(C.c_void_p(x.data_ptr()), C.POINTER(t)) if x is not None else None
    rec = tensors.get("records")
    return abi.tp_cost_tensors(p("node_intra_cost_s"), p("node_intra_volume_bytes"), p("node_memory_bytes"),
                               p("edge_cost_s"), p("edge_volume_bytes"), p("edge_memory_bytes"),
                               C.c_void_p(rec.data_ptr()) if rec is not None else None,
                               p("row_min_cost_s"), p("row_min_volume_bytes"),
                               p("edge_pair_min_cost_s"), p("edge_pair_min_volume_bytes"))


def build_cost_tensors(graph, topo: ClusterTopology, records=False, row_min=False,
                       edge_range=(0, -1), device=-1, pinned=False, pair_form: int = 0) -> CostTensors:
    """The drop-in for build_auxiliary_graph: host graph in, host tensors out
    (a plan built once: on the thread's reused device memory)."""
    plan = Plan(graph, topo, device)
    if pair_form:
        plan.set_pair_form(pair_form)
    return plan.execute_host(records=records, row_min=row_min, edge_range=edge_range, pinned=pinned,
                             scratch=True)


def build_cost_tensors_oneshot(graph, topo: ClusterTopology, device=-1) -> CostTensors:
    """The same build through the one-shot C-ABI call tp_build_cost_tensors
    (the reference-facing entry point; the thread's device memory is reused
    across calls). The output sizes come from a host analysis beforehand."""
    lib = abi.load_engine()
    flat = graph if isinstance(graph, FlatGraph) else flatten(graph)
    plan = Plan(flat, topo, device)
    nn, ne = plan.sizes["num_aux_nodes"], plan.sizes["num_aux_edges"]
    del plan
    n_ops, n_e = flat.num_ops, flat.num_edges
    ix = dict(node_base=np.zeros(n_ops + 1, np.int64), edge_base=np.zeros(n_e + 1, np.int64),
              edge_from_op=np.zeros(max(n_e, 1), np.int32), edge_to_op=np.zeros(max(n_e, 1), np.int32),
              in_degree=np.zeros(max(n_ops, 1), np.int32), out_degree=np.zeros(max(n_ops, 1), np.int32),
              topo_order=np.zeros(max(n_ops, 1), np.int32))
    ct = CostTensors(**ix, **{k: np.zeros(max(nn if k.startswith("node") else ne, 1), np.float64)
                              for k in _OUT_KEYS})
    xi = abi.tp_aux_index(*(abi.ptr(ix[k], C.c_int64 if ix[k].dtype == np.int64 else C.c_int32)
                            for k, _ in abi.tp_aux_index._fields_))
    out = cost_struct(ct)
    gd, td = flat.desc(), topo.desc()
    o = abi.tp_build_opts(0, -1, 0, device, None)
    _check(lib, lib.tp_build_cost_tensors(C.byref(gd), C.byref(td), C.byref(o), C.byref(xi), C.byref(out)))
    for k, m in (("edge_from_op", n_e), ("edge_to_op", n_e), ("in_degree", n_ops), ("out_degree", n_ops),
                 ("topo_order", n_ops)):
        setattr(ct, k, ix[k][:m])
    _trim(ct, nn, ne, 0, 0)
    return ct


def enumerate_strategies(p: int, total_devices: int):
    """Strategy table (layout.hpp:270-328) computed by the device kernel:
    (degrees[S,p], device_map[S,p], matrix_dims[S,p] outermost-first padded
    with 0, matrix_depth[S])."""
    lib = abi.load_engine()
    n = C.c_int64()
    _check(lib, lib.tp_enumerate_strategies(p, total_devices, C.byref(n), None, None, None, None))
    S = n.value
    deg = np.zeros(S * p, np.int64)
    dm = np.zeros(S * p, np.int32)
    md = np.zeros(S * p, np.int64)
    dep = np.zeros(S, np.int32)
    _check(lib, lib.tp_enumerate_strategies(p, total_devices, C.byref(n), abi.ptr(deg, C.c_int64),
                                            abi.ptr(dm, C.c_int32), abi.ptr(md, C.c_int64),
                                            abi.ptr(dep, C.c_int32)))
    return deg.reshape(S, p), dm.reshape(S, p), md.reshape(S, p), dep


def redistribute_batch(queries, form: int = 2):
    """Verification export: each tp_redist_query evaluated by the device
    kernels' pair path (unify + inference + pricing); form 1 = warp per
    pair, 2 = thread per pair."""
    lib = abi.load_engine()
    n = len(queries)
    arr = (abi.tp_redist_query * n)(*queries)
    res = (abi.tp_redist_result * n)()
    _check(lib, lib.tp_redistribute_batch_form(arr, n, res, form))
    return list(res)


_OUT_KEYS = ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes",
             "edge_cost_s", "edge_volume_bytes", "edge_memory_bytes")


class Sweep:
    """A batch of independent (graph, topology) scenarios — cfg5's sweep of
    (model, mesh, bandwidth-ratio) triples — built with the batch entry
    points (tp_plan_create_batch / tp_plan_execute_host_batch): the host
    analysis runs on a pool of host threads and every worker keeps its own
    stream busy, so per-build latencies overlap. Each scenario's result is a
    CostTensors in the reference's index order, exactly what
    build_auxiliary_graph returns for that scenario alone (aux_graph.hpp:211).

    Outputs live in one (optionally pinned) host allocation per tensor kind,
    sliced per scenario, allocated once by `allocate()` and reused by every
    `execute()`."""

    def __init__(self, scenarios, device: int = -1, host_threads: int = 0):
        self.lib = abi.load_engine()
        self.flats = [_flat(g) for g, _ in scenarios]
        self.topos = [t for _, t in scenarios]
        self.device = device
        self.host_threads = host_threads
        n = len(self.flats)
        self._descs = [f.desc() for f in self.flats]
        self._tdescs = [t.desc() for t in self.topos]
        self._gp = (C.POINTER(abi.tp_graph_desc) * max(n, 1))(*[C.pointer(d) for d in self._descs])
        self._tp = (C.POINTER(abi.tp_topology_desc) * max(n, 1))(*[C.pointer(d) for d in self._tdescs])
        self.handles = (C.c_void_p * max(n, 1))()
        self.status = np.zeros(max(n, 1), np.int32)
        self.results = None
        self._outs = None

    def __len__(self):
        return len(self.flats)

    def create(self, raise_errors: bool = True):
        """Host analysis of every scenario (tp_plan_create_batch)."""
        self.destroy()
        st = self.lib.tp_plan_create_batch(self._gp, self._tp, len(self), self.device, self.host_threads,
                                           self.handles, abi.ptr(self.status, C.c_int32))
        if raise_errors:
            _check(self.lib, st)
        return st

    def destroy(self):
        for i in range(len(self)):
            if self.handles[i]:
                self.lib.tp_plan_destroy(self.handles[i])
                self.handles[i] = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def sizes(self, i: int) -> dict:
        s = abi.tp_plan_sizes_t()
        _check(self.lib, self.lib.tp_plan_sizes(self.handles[i], C.byref(s)))
        return {k: getattr(s, k) for k, _ in abi.tp_plan_sizes_t._fields_}

    def allocate(self, pinned: bool = True, records: bool = False, row_min: bool = False):
        """Caller-owned outputs of every scenario (plans must exist). With
        `records` / `row_min` every scenario also gets its AuxEdge records /
        solver minima (cond_min rows and pair_min, both modes); the engine then
        builds the scenarios one execute each instead of one batched launch."""
        n = len(self)
        nn = [self.sizes(i)["num_aux_nodes"] if self.handles[i] else 0 for i in range(n)]
        ne = [self.sizes(i)["num_aux_edges"] if self.handles[i] else 0 for i in range(n)]
        alloc = _pinned_empty if pinned else (lambda k, dt: np.zeros(k, dt))
        node_off = np.concatenate([[0], np.cumsum(nn)]).astype(np.int64)
        edge_off = np.concatenate([[0], np.cumsum(ne)]).astype(np.int64)
        big = {k: alloc(max(int((node_off if k.startswith("node") else edge_off)[-1]), 1), np.float64)
               for k in _OUT_KEYS}
        self._outs = (big, node_off, edge_off)
        self.results = []
        self._cs = (abi.tp_cost_tensors * max(n, 1))()
        self._ix = (abi.tp_aux_index * max(n, 1))()
        self._keep = []
        for i in range(n):
            f = self.flats[i]
            n_ops, n_e = f.num_ops, f.num_edges
            ix = dict(node_base=np.zeros(n_ops + 1, np.int64), edge_base=np.zeros(n_e + 1, np.int64),
                      edge_from_op=np.zeros(max(n_e, 1), np.int32), edge_to_op=np.zeros(max(n_e, 1), np.int32),
                      in_degree=np.zeros(max(n_ops, 1), np.int32), out_degree=np.zeros(max(n_ops, 1), np.int32),
                      topo_order=np.zeros(max(n_ops, 1), np.int32))
            views = {k: big[k][(node_off if k.startswith("node") else edge_off)[i]:
                               (node_off if k.startswith("node") else edge_off)[i + 1]] for k in _OUT_KEYS}
            ct = CostTensors(sizes=self.sizes(i) if self.handles[i] else {}, **ix, **views)
            for k, m in (("edge_from_op", n_e), ("edge_to_op", n_e), ("in_degree", n_ops), ("out_degree", n_ops),
                         ("topo_order", n_ops)):
                setattr(ct, k, ix[k][:m])  # views: filled in place by every execute / build
            if self.handles[i] and records:
                ct.records = np.zeros(max(ne[i], 1) * 40, np.uint8)
            if self.handles[i] and row_min:
                nr = self.sizes(i)["num_rows"]
                ct.row_min_cost_s, ct.row_min_volume_bytes = np.zeros(max(nr, 1)), np.zeros(max(nr, 1))
                ct.edge_pair_min_cost_s = np.zeros(max(f.num_edges, 1))
                ct.edge_pair_min_volume_bytes = np.zeros(max(f.num_edges, 1))
            self.results.append(ct)
            self._cs[i] = cost_struct(ct) if ne[i] + nn[i] > 0 else abi.tp_cost_tensors()
            self._ix[i] = abi.tp_aux_index(*(abi.ptr(ix[k], C.c_int64 if ix[k].dtype == np.int64 else C.c_int32)
                                             for k, _ in abi.tp_aux_index._fields_))
            self._keep.append(ix)
        return self

    def execute(self, raise_errors: bool = True):
        """Build every scenario into its host slices (tp_plan_execute_host_batch)."""
        st = self.lib.tp_plan_execute_host_batch(self.handles, len(self), self._ix, self._cs, self.host_threads,
                                                 abi.ptr(self.status, C.c_int32))
        if raise_errors:
            _check(self.lib, st)
        return st  # the results' index arrays are views set up by allocate()

    def build(self, raise_errors: bool = True):
        """Analyse and build every scenario in one pipelined call
        (tp_build_cost_tensors_batch): the host analysis of one chunk of
        scenarios overlaps the device build of the previous one, and the
        pinned output slices from allocate() are written by the kernels
        directly. Needs allocate() (the output sizes) from an earlier create();
        the plans of that create are not used."""
        st = self.lib.tp_build_cost_tensors_batch(self._gp, self._tp, len(self), self.device, self.host_threads,
                                                  self._ix, self._cs, abi.ptr(self.status, C.c_int32))
        if raise_errors:
            _check(self.lib, st)
        return st  # the results' index arrays are views set up by allocate()

    @property
    def num_aux_edges(self) -> int:
        return int(self._outs[2][-1]) if self._outs else 0


def build_sweep(scenarios, device: int = -1, host_threads: int = 0, pinned: bool = False):
    """Cost tensors of every (graph, topology) scenario: a list of CostTensors,
    element i equal to build_cost_tensors(*scenarios[i])."""
    sw = Sweep(scenarios, device, host_threads)
    sw.create()
    sw.allocate(pinned=pinned)
    sw.execute()
    res = sw.results
    sw.destroy()
    return res


class DeviceSweep:
    """A sweep kept resident on one GPU: every scenario analysed once, its
    descriptors uploaded on its own arena, its cost tensors in slices of one
    device allocation per tensor kind. `run()` rebuilds every scenario with
    ONE persistent launch (tp_plan_execute_batch): the pricing units and the
    output ranges of all scenarios share one work queue, so many small,
    latency-bound builds overlap instead of paying a launch each."""

    def __init__(self, scenarios, device: int = 0):
        import torch
        self.torch = torch
        self.device = device
        self.lib = abi.load_engine()
        self.plans = [Plan(g, t, device=device) for g, t in scenarios]
        n = len(self.plans)
        dev = torch.device("cuda", device)
        self.main = torch.cuda.Stream(dev)
        ne = [p.sizes["num_aux_edges"] for p in self.plans]
        nn = [p.sizes["num_aux_nodes"] for p in self.plans]
        self.edge_off = np.concatenate([[0], np.cumsum(ne)]).astype(np.int64)
        self.node_off = np.concatenate([[0], np.cumsum(nn)]).astype(np.int64)
        self.out = {k: torch.empty(max(int(self.edge_off[-1]), 1), dtype=torch.float64, device=dev)
                    for k in _OUT_KEYS if k.startswith("edge")}
        self.out.update({k: torch.empty(max(int(self.node_off[-1]), 1), dtype=torch.float64, device=dev)
                         for k in _OUT_KEYS if k.startswith("node")})
        self._handles = (C.c_void_p * max(n, 1))(*[p.handle for p in self.plans])
        self._structs = (abi.tp_cost_tensors * max(n, 1))()
        for i, p in enumerate(self.plans):
            p.upload(self.main.cuda_stream)
            sl = self.result(i)
            self._structs[i] = device_cost_struct({k: v for k, v in sl.items() if v.numel()})
        torch.cuda.synchronize(dev)

    @property
    def num_aux_edges(self) -> int:
        return int(self.edge_off[-1])

    @property
    def num_aux_nodes(self) -> int:
        return int(self.node_off[-1])

    def launches_per_run(self) -> int:
        """Kernel launches of the last run: the batch's inference pass and
        build launch(es) (tp_batch_last_launches)."""
        return int(self.lib.tp_batch_last_launches(self.device)) if self.plans else 0

    def set_profile_events(self, start, stop):
        """torch.cuda.Event pair recorded around the batch's kernels of every
        run (tp_batch_set_profile_events); None disables."""
        _check(self.lib, self.lib.tp_batch_set_profile_events(
            self.device, C.c_void_p(start.cuda_event if start is not None else None),
            C.c_void_p(stop.cuda_event if stop is not None else None)))

    def run(self):
        """Rebuild every scenario, asynchronously on `self.main`."""
        _check(self.lib, self.lib.tp_plan_execute_batch(self._handles, len(self.plans), self._structs,
                                                         C.c_void_p(self.main.cuda_stream)))

    def check_errors(self):
        for p in self.plans:
            p.check_errors()

    def result(self, i: int) -> dict:
        """Scenario i's tensors (device slices)."""
        return {k: (v[self.edge_off[i]:self.edge_off[i + 1]] if k.startswith("edge")
                    else v[self.node_off[i]:self.node_off[i + 1]]) for k, v in self.out.items()}
