"""ctypes mirror of include/taps_b200.h (the engine's C-ABI).

The same structs describe the inputs of the engine (libtaps_b200.so) and of
the test-only oracles (oracle/liboracle.so, oracle/_ref/libtopoplan_ref.so),
so a parity test hands the very same descriptor to all three.
"""
from __future__ import annotations

import ctypes as C
import os

# include/taps_b200.h TP_ABI_VERSION this module's struct mirrors follow
TP_ABI_VERSION = 2

TP_OK = 0
TP_ERR_INVALID_ARGUMENT = 1
TP_ERR_TOPOPLAN = 2
TP_ERR_OUT_OF_RANGE = 3
TP_ERR_CUDA = 4
TP_ERR_CAPACITY = 5

TP_MAX_RANK = 8
TP_MAX_AXES = 8
TP_MAX_UNIFIED_DEPTH = 16
TP_MAX_UNIFIED_RANK = 32
TP_MAX_PLAN_OPS = 64

ERROR_KINDS = {
    0: "none", 1: "cycle", 2: "dangling-edge", 3: "devices-not-pow2",
    4: "no-axes", 5: "unknown-slice-tensor", 6: "indivisible-extent",
    7: "shape-mismatch", 8: "not-unifiable", 9: "factorization", 10: "refine",
    11: "device-split", 12: "no-converge", 13: "refine-mismatch",
    14: "deadlock", 15: "no-terminate", 16: "edge-tensor-missing",
    17: "axis-count", 18: "capacity",
}

_p_i32 = C.POINTER(C.c_int32)
_p_i64 = C.POINTER(C.c_int64)
_p_f64 = C.POINTER(C.c_double)


class tp_graph_desc(C.Structure):
    _fields_ = [
        ("num_ops", C.c_int32),
        ("op_id", _p_i32),
        ("op_tensor_begin", _p_i32),
        ("op_num_inputs", _p_i32),
        ("op_axis_begin", _p_i32),
        ("tensor_name", _p_i32),
        ("tensor_shape_begin", _p_i32),
        ("shape", _p_i64),
        ("tensor_element_size", _p_i32),
        ("axis_slice_begin", _p_i32),
        ("slice_tensor", _p_i32),
        ("slice_dim", _p_i32),
        ("num_edges", C.c_int32),
        ("edge_from", _p_i32),
        ("edge_to", _p_i32),
        ("edge_tensor", _p_i32),
    ]


class tp_topology_desc(C.Structure):
    _fields_ = [
        ("node_count", C.c_int32),
        ("local_device_num", C.c_int32),
        ("intra_bandwidth", C.c_double),
        ("inter_bandwidth", C.c_double),
        ("device_memory", C.c_double),
    ]


class tp_aux_index(C.Structure):
    _fields_ = [
        ("node_base", _p_i64),
        ("edge_base", _p_i64),
        ("edge_from_op", _p_i32),
        ("edge_to_op", _p_i32),
        ("in_degree", _p_i32),
        ("out_degree", _p_i32),
        ("topo_order", _p_i32),
    ]


class tp_cost_tensors(C.Structure):
    _fields_ = [
        ("node_intra_cost_s", _p_f64),
        ("node_intra_volume_bytes", _p_f64),
        ("node_memory_bytes", _p_f64),
        ("edge_cost_s", _p_f64),
        ("edge_volume_bytes", _p_f64),
        ("edge_memory_bytes", _p_f64),
        ("aux_edge_records", C.c_void_p),
        ("row_min_cost_s", _p_f64),
        ("row_min_volume_bytes", _p_f64),
        ("edge_pair_min_cost_s", _p_f64),
        ("edge_pair_min_volume_bytes", _p_f64),
    ]


class tp_build_opts(C.Structure):
    _fields_ = [
        ("edge_begin", C.c_int32),
        ("edge_end", C.c_int32),
        ("skip_nodes", C.c_int32),
        ("device", C.c_int32),
        ("stream", C.c_void_p),
    ]


class tp_plan_sizes_t(C.Structure):
    _fields_ = [
        ("num_ops", C.c_int64),
        ("num_edges", C.c_int64),
        ("num_aux_nodes", C.c_int64),
        ("num_aux_edges", C.c_int64),
        ("num_virtual_edges", C.c_int64),
        ("num_rows", C.c_int64),
        ("num_signatures", C.c_int64),
        ("num_pair_evals", C.c_int64),
        ("h2d_bytes", C.c_int64),
        ("num_class_rows", C.c_int64),
        ("num_pair_slots", C.c_int64),
    ]


class tp_redist_query(C.Structure):
    _fields_ = [
        ("rank", C.c_int32),
        ("shape", _p_i64),
        ("from_depth", C.c_int32),
        ("from_dims", _p_i64),
        ("from_map", _p_i32),
        ("to_depth", C.c_int32),
        ("to_dims", _p_i64),
        ("to_map", _p_i32),
        ("tensor_bytes", C.c_double),
        ("local_device_num", C.c_int32),
        ("intra_bandwidth", C.c_double),
        ("inter_bandwidth", C.c_double),
    ]


class tp_redist_result(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("depth", C.c_int32),
        ("dims", C.c_int64 * TP_MAX_UNIFIED_DEPTH),
        ("urank", C.c_int32),
        ("shape", C.c_int64 * TP_MAX_UNIFIED_RANK),
        ("from_map", C.c_int32 * TP_MAX_UNIFIED_RANK),
        ("to_map", C.c_int32 * TP_MAX_UNIFIED_RANK),
        ("num_ops", C.c_int32),
        ("ops", (C.c_int32 * 5) * TP_MAX_PLAN_OPS),
        ("op_ct", C.c_int64 * TP_MAX_PLAN_OPS),
        ("op_seconds", C.c_double * TP_MAX_PLAN_OPS),
        ("volume_bytes", C.c_double),
        ("seconds", C.c_double),
    ]

    def plan(self):
        """(unified dims, shape, from_map, to_map, ops, cts) as plain tuples."""
        n = self.num_ops
        return (
            tuple(self.dims[: self.depth]),
            tuple(self.shape[: self.urank]),
            tuple(self.from_map[: self.urank]),
            tuple(self.to_map[: self.urank]),
            tuple(tuple(self.ops[i]) for i in range(n)),
            tuple(self.op_ct[i] for i in range(n)),
        )


def ptr(arr, ctype):
    """ctypes pointer to a numpy array's data (None for None)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(C.POINTER(ctype))


PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
ENGINE_SO = os.path.join(PKG_DIR, "libtaps_b200.so")


class EngineMissing(RuntimeError):
    pass


_engine = None


def load_engine() -> C.CDLL:
    """Load the CUDA engine. There is no CPU fallback: a missing library is
    an error, never a silent switch to another implementation."""
    global _engine
    if _engine is not None:
        return _engine
    if not os.path.exists(ENGINE_SO):
        raise EngineMissing(
            f"{ENGINE_SO} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = C.CDLL(ENGINE_SO)
    P = C.POINTER
    lib.tp_build_cost_tensors.argtypes = [P(tp_graph_desc), P(tp_topology_desc), P(tp_build_opts),
                                          P(tp_aux_index), P(tp_cost_tensors)]
    lib.tp_build_cost_tensors.restype = C.c_int
    lib.tp_plan_create.argtypes = [P(tp_graph_desc), P(tp_topology_desc), C.c_int32, P(C.c_void_p)]
    lib.tp_plan_create.restype = C.c_int
    lib.tp_plan_destroy.argtypes = [C.c_void_p]
    lib.tp_plan_destroy.restype = None
    lib.tp_plan_sizes.argtypes = [C.c_void_p, P(tp_plan_sizes_t)]
    lib.tp_plan_sizes.restype = C.c_int
    lib.tp_plan_index.argtypes = [C.c_void_p, P(tp_aux_index)]
    lib.tp_plan_index.restype = C.c_int
    lib.tp_plan_upload.argtypes = [C.c_void_p, C.c_void_p]
    lib.tp_plan_upload.restype = C.c_int
    lib.tp_plan_execute.argtypes = [C.c_void_p, P(tp_build_opts), P(tp_cost_tensors)]
    lib.tp_plan_execute.restype = C.c_int
    lib.tp_plan_execute_host.argtypes = [C.c_void_p, P(tp_build_opts), P(tp_aux_index), P(tp_cost_tensors)]
    lib.tp_plan_execute_host.restype = C.c_int
    lib.tp_plan_execute_host_scratch.argtypes = [C.c_void_p, P(tp_build_opts), P(tp_aux_index), P(tp_cost_tensors)]
    lib.tp_plan_execute_host_scratch.restype = C.c_int
    lib.tp_plan_check_errors.argtypes = [C.c_void_p]
    lib.tp_plan_check_errors.restype = C.c_int
    lib.tp_plan_set_profile_events.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.tp_plan_set_profile_events.restype = C.c_int
    lib.tp_plan_set_timeline.argtypes = [C.c_void_p, C.c_int32]
    lib.tp_plan_set_timeline.restype = C.c_int
    lib.tp_plan_timeline.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    lib.tp_plan_timeline.restype = C.c_int
    lib.tp_plan_timeline_detail.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_uint32),
                                            C.POINTER(C.c_int64)]
    lib.tp_plan_timeline_detail.restype = C.c_int
    lib.tp_plan_last_launches.argtypes = [C.c_void_p]
    lib.tp_plan_last_launches.restype = C.c_int64
    lib.tp_enumerate_strategies.argtypes = [C.c_int32, C.c_int64, P(C.c_int64), _p_i64, _p_i32,
                                            _p_i64, _p_i32]
    lib.tp_enumerate_strategies.restype = C.c_int
    lib.tp_redistribute_batch.argtypes = [P(tp_redist_query), C.c_int32, P(tp_redist_result)]
    lib.tp_redistribute_batch.restype = C.c_int
    lib.tp_redistribute_batch_form.argtypes = [P(tp_redist_query), C.c_int32, P(tp_redist_result), C.c_int32]
    lib.tp_redistribute_batch_form.restype = C.c_int
    lib.tp_plan_set_pair_form.argtypes = [C.c_void_p, C.c_int32]
    lib.tp_plan_set_pair_form.restype = C.c_int
    lib.tp_plan_create_batch.argtypes = [P(P(tp_graph_desc)), P(P(tp_topology_desc)), C.c_int32, C.c_int32,
                                         C.c_int32, P(C.c_void_p), _p_i32]
    lib.tp_plan_create_batch.restype = C.c_int
    lib.tp_plan_execute_host_batch.argtypes = [P(C.c_void_p), C.c_int32, P(tp_aux_index), P(tp_cost_tensors),
                                               C.c_int32, _p_i32]
    lib.tp_plan_execute_host_batch.restype = C.c_int
    lib.tp_plan_execute_batch.argtypes = [P(C.c_void_p), C.c_int32, P(tp_cost_tensors), C.c_void_p]
    lib.tp_plan_execute_batch.restype = C.c_int
    lib.tp_plan_price_assignments.argtypes = [C.c_void_p, P(tp_cost_tensors), _p_i32, C.c_int32, P(C.c_double),
                                              P(C.c_double), P(C.c_double), C.c_void_p]
    lib.tp_plan_price_assignments.restype = C.c_int
    lib.tp_build_cost_tensors_batch.argtypes = [P(P(tp_graph_desc)), P(P(tp_topology_desc)), C.c_int32, C.c_int32,
                                                C.c_int32, P(tp_aux_index), P(tp_cost_tensors), _p_i32]
    lib.tp_build_cost_tensors_batch.restype = C.c_int
    lib.tp_plan_export_lp.argtypes = [C.c_void_p, P(tp_cost_tensors), C.c_int32, C.c_double, C.c_char_p,
                                      P(C.c_int64)]
    lib.tp_plan_export_lp.restype = C.c_int
    lib.tp_batch_set_profile_events.argtypes = [C.c_int32, C.c_void_p, C.c_void_p]
    lib.tp_batch_set_profile_events.restype = C.c_int
    lib.tp_batch_last_launches.argtypes = [C.c_int32]
    lib.tp_batch_last_launches.restype = C.c_int64
    lib.tp_build_cost_tensors_multi.argtypes = [P(tp_graph_desc), P(tp_topology_desc), _p_i32, C.c_int32,
                                                P(tp_aux_index), P(tp_cost_tensors)]
    lib.tp_build_cost_tensors_multi.restype = C.c_int
    lib.tp_plan_execute_host_multi.argtypes = [C.c_void_p, _p_i32, C.c_int32, P(tp_aux_index), P(tp_cost_tensors)]
    lib.tp_plan_execute_host_multi.restype = C.c_int
    lib.tp_plan_set_bandwidth.argtypes = [C.c_void_p, C.c_double, C.c_double]
    lib.tp_plan_set_bandwidth.restype = C.c_int
    lib.tp_last_error.argtypes = []
    lib.tp_last_error.restype = C.c_char_p
    lib.tp_last_error_kind.argtypes = []
    lib.tp_last_error_kind.restype = C.c_int32
    lib.tp_abi_version.argtypes = []
    lib.tp_abi_version.restype = C.c_int32
    if lib.tp_abi_version() != TP_ABI_VERSION:  # a stale build would read the structs wrong
        raise EngineMissing(f"{ENGINE_SO} has ABI version {lib.tp_abi_version()}, expected {TP_ABI_VERSION}; rebuild it")
    _engine = lib
    return lib


# Every symbol include/taps_b200.h declares (checked by the CPU test suite).
EXPORTED_SYMBOLS = (
    "tp_build_cost_tensors", "tp_plan_create", "tp_plan_destroy", "tp_plan_sizes",
    "tp_plan_index", "tp_plan_upload", "tp_plan_execute", "tp_plan_execute_host", "tp_plan_execute_host_scratch", "tp_plan_check_errors",
    "tp_plan_last_launches", "tp_plan_set_profile_events", "tp_plan_set_timeline", "tp_plan_timeline", "tp_plan_timeline_detail", "tp_enumerate_strategies", "tp_redistribute_batch",
    "tp_redistribute_batch_form", "tp_plan_set_pair_form", "tp_plan_create_batch", "tp_plan_execute_host_batch",
    "tp_plan_execute_batch", "tp_plan_price_assignments", "tp_plan_set_bandwidth",
    "tp_build_cost_tensors_multi", "tp_plan_execute_host_multi", "tp_batch_last_launches",
    "tp_plan_export_lp", "tp_build_cost_tensors_batch",
    "tp_batch_set_profile_events",
    "tp_last_error", "tp_last_error_kind", "tp_abi_version",
)


class TopoplanError(RuntimeError):
    """Mirror of topoplan::Error (validation.hpp:29-32)."""


def raise_for_status(status: int, message: str = "", kind: int = 0):
    if status == TP_OK:
        return
    text = f"{message} [{ERROR_KINDS.get(kind, kind)}]" if message else ERROR_KINDS.get(kind, str(kind))
    if status == TP_ERR_TOPOPLAN:
        raise TopoplanError(text)
    if status == TP_ERR_OUT_OF_RANGE:
        raise IndexError(text)  # std::out_of_range
    if status == TP_ERR_CAPACITY:
        raise OverflowError(text)
    if status == TP_ERR_CUDA:
        raise RuntimeError("CUDA: " + text)
    raise ValueError(text)
