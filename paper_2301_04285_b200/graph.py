"""Host-side input types of the cost-tensor build, mirroring the reference's
topoplan::TensorSpec / OperatorNode / ComputationGraph / ClusterTopology
(/root/reference/proj/include/topoplan/graph.hpp:39-351) with the same
field names, plus `flatten()` which produces the C-ABI descriptor
(include/taps_b200.h, tp_graph_desc).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import abi


def is_power_of_two(n: int) -> bool:  # graph.hpp:115
    return n > 0 and (n & (n - 1)) == 0


@dataclass
class TensorSpec:  # graph.hpp:39-60
    name: str
    shape: List[int]
    element_size: int = 4

    def rank(self) -> int:
        return len(self.shape)

    def elements(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n

    def bytes(self) -> float:
        return float(self.elements()) * self.element_size


@dataclass
class AxisSlice:  # graph.hpp:84-90
    tensor: str
    dim: int = 0


@dataclass
class OperatorAxis:  # graph.hpp:91-94
    name: str
    slices: List[AxisSlice] = field(default_factory=list)


@dataclass
class OperatorNode:  # graph.hpp:96-123
    id: str
    kind: str = "other"  # matmul | conv | elementwise | other (graph.hpp:62-80)
    inputs: List[TensorSpec] = field(default_factory=list)
    outputs: List[TensorSpec] = field(default_factory=list)
    axes: List[OperatorAxis] = field(default_factory=list)

    def axis_count(self) -> int:
        return len(self.axes)

    def find_input(self, name):
        return next((t for t in self.inputs if t.name == name), None)

    def find_output(self, name):
        return next((t for t in self.outputs if t.name == name), None)

    def find_tensor(self, name):
        return self.find_input(name) or self.find_output(name)


@dataclass
class GraphEdge:  # graph.hpp:125-129
    from_: str
    to: str
    tensor: str


@dataclass
class ComputationGraph:  # graph.hpp:131-184
    operators: List[OperatorNode] = field(default_factory=list)
    edges: List[GraphEdge] = field(default_factory=list)

    def find_op(self, id: str) -> int:
        # first operator with the id, like the reference's linear scan
        # (graph.hpp:135-140), but indexed
        idx = self.__dict__.get("_find_cache")
        if idx is None or idx[0] != len(self.operators):
            table: Dict[str, int] = {}
            for i, op in enumerate(self.operators):
                table.setdefault(op.id, i)
            idx = (len(self.operators), table)
            self.__dict__["_find_cache"] = idx
        return idx[1].get(id, -1)

    def in_degree(self, i: int) -> int:
        return sum(1 for e in self.edges if e.to == self.operators[i].id)

    def out_degree(self, i: int) -> int:
        return sum(1 for e in self.edges if e.from_ == self.operators[i].id)

    def topological_order(self) -> List[int]:  # Kahn, graph.hpp:158-183
        n = len(self.operators)
        indeg = [0] * n
        succ: List[List[int]] = [[] for _ in range(n)]
        for e in self.edges:
            u, w = self.find_op(e.from_), self.find_op(e.to)
            if u < 0 or w < 0:
                continue
            succ[u].append(w)
            indeg[w] += 1
        ready = [i for i in range(n) if indeg[i] == 0]
        order = []
        head = 0
        while head < len(ready):
            u = ready[head]
            head += 1
            order.append(u)
            for w in succ[u]:
                indeg[w] -= 1
                if indeg[w] == 0:
                    ready.append(w)
        return order if len(order) == n else []


@dataclass
class ClusterTopology:  # graph.hpp:189-199
    node_count: int = 1
    local_device_num: int = 1
    intra_bandwidth: float = 0.0  # bytes/s
    inter_bandwidth: float = 0.0  # bytes/s
    device_memory: float = 0.0  # bytes

    def total_devices(self) -> int:
        return self.node_count * self.local_device_num

    def desc(self) -> abi.tp_topology_desc:
        return abi.tp_topology_desc(self.node_count, self.local_device_num, self.intra_bandwidth,
                                    self.inter_bandwidth, self.device_memory)


# --------------------------------------------------------------------------
# validation: graph.hpp:201-351 (ValidationReport, validation.hpp:41-82)
# --------------------------------------------------------------------------

@dataclass
class Issue:
    severity: str  # "error" | "warning"
    code: str
    message: str


@dataclass
class ValidationReport:
    issues: List[Issue] = field(default_factory=list)

    def ok(self) -> bool:
        return not any(i.severity == "error" for i in self.issues)

    def has(self, code: str) -> bool:
        return any(i.code == code for i in self.issues)

    def add_error(self, code, message):
        self.issues.append(Issue("error", code, message))

    def add_warning(self, code, message):
        self.issues.append(Issue("warning", code, message))


def validate_topology(topo: ClusterTopology) -> ValidationReport:  # graph.hpp:201-233
    r = ValidationReport()
    if topo.node_count < 1:
        r.add_error("node-count", "node_count must be >= 1")
    if topo.local_device_num < 1:
        r.add_error("local-device-num", "local_device_num must be >= 1")
    if topo.node_count >= 1 and topo.local_device_num >= 1:
        if not is_power_of_two(topo.local_device_num):
            r.add_error("power-of-two", f"local_device_num {topo.local_device_num} is not a power of two")
        if not is_power_of_two(topo.total_devices()):
            r.add_error("power-of-two", f"total device count {topo.total_devices()} is not a power of two")
    if topo.intra_bandwidth <= 0 or topo.inter_bandwidth <= 0:
        r.add_error("bandwidth", "bandwidths must be positive")
    elif topo.inter_bandwidth > topo.intra_bandwidth:
        r.add_warning("bandwidth-order", "inter-node bandwidth exceeds intra-node bandwidth")
    if topo.device_memory <= 0:
        r.add_error("device-memory", "device_memory must be positive")
    return r


def validate_graph(graph: ComputationGraph) -> ValidationReport:  # graph.hpp:235-351
    r = ValidationReport()
    ids = set()
    for op in graph.operators:
        if op.id in ids:
            r.add_error("duplicate-id", f"duplicate operator id '{op.id}'")
        ids.add(op.id)
    for op in graph.operators:
        for t in op.inputs + op.outputs:
            if any(s < 1 for s in t.shape):
                r.add_error("bad-extent", f"tensor '{t.name}' of operator '{op.id}' has extent < 1")
            if t.element_size not in (1, 2, 4, 8):
                r.add_error("element-size", f"tensor '{t.name}' of operator '{op.id}' has element_size outside {{1,2,4,8}}")
        if not op.axes:
            r.add_error("no-axes", f"operator '{op.id}' declares no partitionable axes")
        names = set()
        for axis in op.axes:
            if axis.name in names:
                r.add_error("duplicate-axis", f"operator '{op.id}' repeats axis '{axis.name}'")
            names.add(axis.name)
            if not axis.slices:
                r.add_error("axis-no-slice", f"axis '{axis.name}' of operator '{op.id}' maps to no tensor dimension")
            for s in axis.slices:
                t = op.find_tensor(s.tensor)
                if t is None:
                    r.add_error("dangling-reference", f"axis '{axis.name}' of operator '{op.id}' references unknown tensor '{s.tensor}'")
                elif s.dim < 0 or s.dim >= t.rank():
                    r.add_error("axis-bad-dim", f"axis '{axis.name}' of operator '{op.id}' references dimension {s.dim} of tensor '{s.tensor}'")
        sliced = set()
        for axis in op.axes:
            for s in axis.slices:
                if (s.tensor, s.dim) in sliced:
                    r.add_error("dim-double-sliced", f"operator '{op.id}' slices tensor '{s.tensor}' dimension {s.dim} with more than one axis")
                sliced.add((s.tensor, s.dim))
    for e in graph.edges:
        u, w = graph.find_op(e.from_), graph.find_op(e.to)
        if u < 0:
            r.add_error("dangling-reference", f"edge references missing operator '{e.from_}'")
        if w < 0:
            r.add_error("dangling-reference", f"edge references missing operator '{e.to}'")
        if u < 0 or w < 0:
            continue
        produced = graph.operators[u].find_output(e.tensor)
        consumed = graph.operators[w].find_input(e.tensor)
        if produced is None:
            r.add_error("dangling-reference", f"operator '{e.from_}' has no output tensor '{e.tensor}'")
        if consumed is None:
            r.add_error("dangling-reference", f"operator '{e.to}' has no input tensor '{e.tensor}'")
        if produced is not None and consumed is not None and (
                produced.shape != consumed.shape or produced.element_size != consumed.element_size):
            r.add_error("shape-mismatch", f"tensor '{e.tensor}' differs between '{e.from_}' and '{e.to}'")
    if not r.has("dangling-reference") and graph.operators and not graph.topological_order():
        r.add_error("cycle", "computation graph contains a cycle")
    return r


# --------------------------------------------------------------------------
# flattening into the C-ABI descriptor
# --------------------------------------------------------------------------

class FlatGraph:
    """Interned, CSR-flattened graph. Keeps the numpy buffers alive for as
    long as the ctypes descriptor is in use."""

    def __init__(self, graph: ComputationGraph):
        op_ids: Dict[str, int] = {}
        names: Dict[str, int] = {}

        def oid(s):
            return op_ids.setdefault(s, len(op_ids))

        def nid(s):
            return names.setdefault(s, len(names))

        op_id, op_tb, op_nin, op_ab = [], [0], [], [0]
        t_name, t_sb, shape, t_es = [], [0], [], []
        a_sb, s_t, s_d = [0], [], []
        for op in graph.operators:
            op_id.append(oid(op.id))
            for t in list(op.inputs) + list(op.outputs):
                t_name.append(nid(t.name))
                shape.extend(int(x) for x in t.shape)
                t_sb.append(len(shape))
                t_es.append(int(t.element_size))
            op_tb.append(len(t_name))
            op_nin.append(len(op.inputs))
            for ax in op.axes:
                for s in ax.slices:
                    s_t.append(nid(s.tensor))
                    s_d.append(int(s.dim))
                a_sb.append(len(s_t))
            op_ab.append(len(a_sb) - 1)
        e_f = [oid(e.from_) for e in graph.edges]
        e_t = [oid(e.to) for e in graph.edges]
        e_n = [nid(e.tensor) for e in graph.edges]

        i32 = lambda v: np.ascontiguousarray(np.asarray(v, dtype=np.int32).reshape(-1))
        self.op_id = i32(op_id)
        self.op_tensor_begin = i32(op_tb)
        self.op_num_inputs = i32(op_nin)
        self.op_axis_begin = i32(op_ab)
        self.tensor_name = i32(t_name)
        self.tensor_shape_begin = i32(t_sb)
        self.shape = np.ascontiguousarray(np.asarray(shape, dtype=np.int64).reshape(-1))
        self.tensor_element_size = i32(t_es)
        self.axis_slice_begin = i32(a_sb)
        self.slice_tensor = i32(s_t)
        self.slice_dim = i32(s_d)
        self.edge_from = i32(e_f)
        self.edge_to = i32(e_t)
        self.edge_tensor = i32(e_n)
        self.num_ops = len(graph.operators)
        self.num_edges = len(graph.edges)
        self.op_ids = op_ids
        self.names = names
        # the empty arrays still need a valid pointer
        for k, v in list(self.__dict__.items()):
            if isinstance(v, np.ndarray) and v.size == 0:
                setattr(self, k, np.zeros(1, dtype=v.dtype))

    def desc(self) -> abi.tp_graph_desc:
        P32 = lambda a: abi.ptr(a, C.c_int32)
        return abi.tp_graph_desc(
            self.num_ops, P32(self.op_id), P32(self.op_tensor_begin), P32(self.op_num_inputs),
            P32(self.op_axis_begin), P32(self.tensor_name), P32(self.tensor_shape_begin),
            abi.ptr(self.shape, C.c_int64), P32(self.tensor_element_size),
            P32(self.axis_slice_begin), P32(self.slice_tensor), P32(self.slice_dim),
            self.num_edges, P32(self.edge_from), P32(self.edge_to), P32(self.edge_tensor))

    def nbytes(self) -> int:
        return sum(v.nbytes for v in self.__dict__.values() if isinstance(v, np.ndarray))


def flatten(graph: ComputationGraph) -> FlatGraph:
    return FlatGraph(graph)
