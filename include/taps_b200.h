/*
 * taps_b200.h — C-ABI of the B200-native TAPS cost-tensor engine.
 *
 * Drop-in boundary for the reference's hot path
 *   topoplan::build_auxiliary_graph(graph, topo, mode)
 *   (/root/reference/proj/include/topoplan/aux_graph.hpp:211-315)
 * The reference is a header-only C++ API with no FFI; this header is the
 * flattened, C-callable form of that one call plus the split
 * plan/execute entry points a multi-GPU or batched caller needs. A header-only
 * C++ adapter (include/taps_b200/aux_graph_b200.hpp) rebuilds the reference's
 * topoplan::AuxiliaryGraph from these arrays so formulate()/solve() run
 * unchanged (solver.hpp:69-176, 417-493).
 *
 * Conventions
 *  - Plain pointers and sizes only; no CUDA or torch types. Streams are
 *    passed as `void*` (a cudaStream_t).
 *  - Strings of the reference (operator ids, tensor names) are interned to
 *    int32 ids by the caller; equality of ids == equality of strings.
 *  - No exceptions cross the ABI. Every entry point returns tp_status; the
 *    message of the last failure on the calling thread is tp_last_error().
 *  - Index conventions are the reference's (aux_graph.hpp:236-296):
 *      aux node id  = node_base[op] + strategy index
 *      aux edge id  = edge_base[e] + su * S(to_op) + sw
 */
#ifndef TAPS_B200_H_
#define TAPS_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 2: tp_cost_tensors gained edge_pair_min_cost_s / edge_pair_min_volume_bytes (appended). */
#define TP_ABI_VERSION 2

typedef enum tp_status {
  TP_OK = 0,
  /* Malformed descriptor (null pointer, broken CSR offsets). */
  TP_ERR_INVALID_ARGUMENT = 1,
  /* A condition on which the reference throws topoplan::Error
     (validation.hpp:29-32): cycle, dangling edge, non-power-of-two device
     count, operator without axes, indivisible extent, non-unifiable layouts,
     redistribution deadlock / non-termination. */
  TP_ERR_TOPOPLAN = 2,
  /* The reference throws std::out_of_range: an edge names a tensor that one
     of its endpoints does not carry (aux_graph.hpp:281,284 `layouts.at`). */
  TP_ERR_OUT_OF_RANGE = 3,
  /* CUDA runtime failure, or no CUDA device (the engine has no CPU path). */
  TP_ERR_CUDA = 4,
  /* Input exceeds a fixed kernel bound (see TP_MAX_*). The reference would
     not fail here; the engine refuses rather than truncate. */
  TP_ERR_CAPACITY = 5,
} tp_status;

/* Which reference condition produced TP_ERR_TOPOPLAN / TP_ERR_OUT_OF_RANGE. */
typedef enum tp_error_kind {
  TP_E_NONE = 0,
  TP_E_CYCLE = 1,               /* aux_graph.hpp:224-226 */
  TP_E_DANGLING_EDGE = 2,       /* aux_graph.hpp:278 */
  TP_E_DEVICES_NOT_POW2 = 3,    /* layout.hpp:272-274 */
  TP_E_NO_AXES = 4,             /* layout.hpp:276 */
  TP_E_UNKNOWN_SLICE_TENSOR = 5,/* layout.hpp:353-356 */
  TP_E_INDIVISIBLE_EXTENT = 6,  /* layout.hpp:359-365 */
  TP_E_SHAPE_MISMATCH = 7,      /* redistribution.hpp:261-263 */
  TP_E_NOT_UNIFIABLE = 8,       /* redistribution.hpp:141, 286 */
  TP_E_FACTORIZATION = 9,       /* redistribution.hpp:102-111 */
  TP_E_REFINE = 10,             /* redistribution.hpp:178-179, 213-214 */
  TP_E_DEVICE_SPLIT = 11,       /* redistribution.hpp:240-241 */
  TP_E_NO_CONVERGE = 12,        /* redistribution.hpp:299 */
  TP_E_REFINE_MISMATCH = 13,    /* redistribution.hpp:333-338 */
  TP_E_DEADLOCK = 14,           /* redistribution.hpp:416 */
  TP_E_NO_TERMINATE = 15,       /* redistribution.hpp:432 */
  TP_E_EDGE_TENSOR_MISSING = 16,/* std::out_of_range, aux_graph.hpp:281,284 */
  TP_E_AXIS_COUNT = 17,         /* layout.hpp:335-336 (cannot occur via build) */
  TP_E_CAPACITY = 18
} tp_error_kind;

/* Fixed bounds of the device kernels (per-thread register/local arrays). */
#define TP_MAX_RANK 8          /* tensor rank */
#define TP_MAX_AXES 8          /* partitionable axes per operator */
#define TP_MAX_LOG2_DEVICES 16 /* total devices <= 65536 */

/* Flattened topoplan::ComputationGraph (graph.hpp:96-184).
 * CSR layout: operator i owns tensors [op_tensor_begin[i], op_tensor_begin[i+1]),
 * the first op_num_inputs[i] of which are its inputs in declaration order
 * (OperatorNode::inputs), the rest its outputs; axes
 * [op_axis_begin[i], op_axis_begin[i+1]) in declaration order; axis a owns
 * slices [axis_slice_begin[a], axis_slice_begin[a+1]). */
typedef struct tp_graph_desc {
  int32_t num_ops;
  const int32_t* op_id;              /* [num_ops] interned OperatorNode::id  */
  const int32_t* op_tensor_begin;    /* [num_ops + 1]                         */
  const int32_t* op_num_inputs;      /* [num_ops]                             */
  const int32_t* op_axis_begin;      /* [num_ops + 1]                         */
  const int32_t* tensor_name;        /* [num_tensors] interned TensorSpec::name */
  const int32_t* tensor_shape_begin; /* [num_tensors + 1] CSR into shape      */
  const int64_t* shape;              /* extents, TensorSpec::shape            */
  const int32_t* tensor_element_size;/* [num_tensors]                         */
  const int32_t* axis_slice_begin;   /* [num_axes + 1]                        */
  const int32_t* slice_tensor;       /* [num_slices] interned AxisSlice::tensor */
  const int32_t* slice_dim;          /* [num_slices] AxisSlice::dim           */
  int32_t num_edges;
  const int32_t* edge_from;          /* [num_edges] interned GraphEdge::from  */
  const int32_t* edge_to;            /* [num_edges] interned GraphEdge::to    */
  const int32_t* edge_tensor;        /* [num_edges] interned GraphEdge::tensor */
} tp_graph_desc;

/* topoplan::ClusterTopology (graph.hpp:189-199); bandwidths in bytes/s. */
typedef struct tp_topology_desc {
  int32_t node_count;
  int32_t local_device_num;
  double intra_bandwidth;
  double inter_bandwidth;
  double device_memory;
} tp_topology_desc;

/* Index structure of the auxiliary graph; all arrays caller-owned and
 * optional (NULL skips). Sizes come from tp_plan_sizes(). */
typedef struct tp_aux_index {
  int64_t* node_base;    /* [num_ops + 1]   first aux node of each operator   */
  int64_t* edge_base;    /* [num_edges + 1] first aux edge of each graph edge */
  int32_t* edge_from_op; /* [num_edges]     find_op(from)                     */
  int32_t* edge_to_op;   /* [num_edges]     find_op(to)                       */
  int32_t* in_degree;    /* [num_ops]       ComputationGraph::in_degree       */
  int32_t* out_degree;   /* [num_ops]       ComputationGraph::out_degree      */
  int32_t* topo_order;   /* [num_ops]       ComputationGraph::topological_order */
} tp_aux_index;

/* Cost tensors, structure of arrays, fp64 (aux_graph.hpp:42-59).
 * Pointers are caller-owned, either all device pointers (tp_plan_execute) or
 * all host pointers (tp_build_cost_tensors; pinned memory recommended).
 * Any pointer may be NULL to skip that tensor. */
typedef struct tp_cost_tensors {
  double* node_intra_cost_s;       /* [num_aux_nodes] AuxNode::intra_cost_s       */
  double* node_intra_volume_bytes; /* [num_aux_nodes] AuxNode::intra_volume_bytes */
  double* node_memory_bytes;       /* [num_aux_nodes] AuxNode::memory_bytes       */
  double* edge_cost_s;             /* [num_aux_edges] AuxEdge::cost_s             */
  double* edge_volume_bytes;       /* [num_aux_edges] AuxEdge::volume_bytes       */
  double* edge_memory_bytes;       /* [num_aux_edges] AuxEdge::memory_bytes       */
  /* Optional AoS export with the exact memory layout of topoplan::AuxEdge
   * {int original_edge, from_node, to_node; double cost_s, volume_bytes,
   *  memory_bytes} (40 bytes, aux_graph.hpp:52-59): NULL skips. */
  void* aux_edge_records;          /* [num_aux_edges * 40 bytes]                  */
  /* Optional per-(edge, src strategy) row minima of the edge weight, the
   * solver's cond_min (solver.hpp:239-253), for both cost modes. */
  double* row_min_cost_s;          /* [num_rows] */
  double* row_min_volume_bytes;    /* [num_rows] */
  /* Optional per-graph-edge minimum over its rows, the solver's pair_min
   * (solver.hpp:254-255), both cost modes. Requires the row minima above
   * (TP_ERR_INVALID_ARGUMENT otherwise). */
  double* edge_pair_min_cost_s;       /* [num_edges of the slice] */
  double* edge_pair_min_volume_bytes; /* [num_edges of the slice] */
} tp_cost_tensors;

typedef struct tp_build_opts {
  /* Build only graph edges [edge_begin, edge_end) (aux edges
   * [edge_base[edge_begin], edge_base[edge_end])). Output pointers then index
   * that slice from 0. edge_end < 0 means num_edges. */
  int32_t edge_begin;
  int32_t edge_end;
  /* Skip the per-node tensors (another shard writes them). */
  int32_t skip_nodes;
  int32_t device;    /* CUDA device ordinal; -1 = current */
  void* stream;      /* cudaStream_t; NULL = the per-plan stream */
} tp_build_opts;

typedef struct tp_plan tp_plan; /* opaque */

typedef struct tp_plan_sizes_t {
  int64_t num_ops;
  int64_t num_edges;
  int64_t num_aux_nodes;
  int64_t num_aux_edges;
  int64_t num_virtual_edges;
  int64_t num_rows;          /* sum over edges of S(from op) */
  int64_t num_signatures;    /* distinct edge classes priced */
  int64_t num_pair_evals;    /* (signature, su, sw) pairs priced on device */
  int64_t h2d_bytes;         /* descriptor bytes copied to the device */
  int64_t num_class_rows;    /* node-class strategy rows priced on device */
  int64_t num_pair_slots;    /* strategy pairs of the distinct edge classes; num_pair_evals is
                                smaller where classes share layouts or derive from another */
} tp_plan_sizes_t;

/* --- one-shot call: the drop-in for build_auxiliary_graph ---------------- */

/* Host in, host out (pinned recommended): validates like the reference,
 * uploads the descriptors, runs the kernels, copies the cost tensors back. */
tp_status tp_build_cost_tensors(const tp_graph_desc* graph,
                                const tp_topology_desc* topo,
                                const tp_build_opts* opts,
                                tp_aux_index* index_out,
                                tp_cost_tensors* host_out);

/* Single-process multi-GPU form of the one-shot call: the
 * graph's edges are cut into contiguous ranges balanced by their aux-edge
 * counts sum |Su| x |Sw|; devices[i] builds range i (devices[0] also the
 * per-node tensors) and copies its slice [edge_base[e0], edge_base[e1]) of
 * every requested edge tensor -- SoA, AuxEdge records, row / pair minima --
 * straight into host_out at that offset (aux_graph.hpp:93-98, 273-296). No
 * collective: the ranges are independent. Results equal tp_build_cost_tensors
 * bit for bit; errors are the reference's first (the smallest over devices). */
tp_status tp_build_cost_tensors_multi(const tp_graph_desc* graph,
                                      const tp_topology_desc* topo,
                                      const int32_t* devices, int32_t num_devices,
                                      tp_aux_index* index_out,
                                      tp_cost_tensors* host_out);

/* --- split API: analyse once, execute on device-resident buffers --------- */

tp_status tp_plan_create(const tp_graph_desc* graph,
                         const tp_topology_desc* topo, int32_t device,
                         tp_plan** plan_out);
void tp_plan_destroy(tp_plan* plan);
tp_status tp_plan_sizes(const tp_plan* plan, tp_plan_sizes_t* sizes);
tp_status tp_plan_index(const tp_plan* plan, tp_aux_index* index_out);
/* Upload the plan's descriptors (tables, signatures) to the device. */
tp_status tp_plan_upload(tp_plan* plan, void* stream);
/* Run the kernels into DEVICE pointers. Asynchronous on `stream`; errors
 * detected by the kernels are reported by tp_plan_check_errors(). */
tp_status tp_plan_execute(tp_plan* plan, const tp_build_opts* opts,
                          tp_cost_tensors* device_out);
/* Run the kernels and copy the requested tensors back into HOST pointers
 * (the one-shot call on an existing plan; synchronous). */
tp_status tp_plan_execute_host(tp_plan* plan, const tp_build_opts* opts,
                               tp_aux_index* index_out, tp_cost_tensors* host_out);
/* tp_plan_execute_host on the calling thread's scratch device memory (the
 * buffers tp_build_cost_tensors reuses across calls) instead of the plan's
 * own: no device allocation or release when the thread built a graph of the
 * same sizes before, and the plan keeps no device state afterwards (a plan
 * that already has its own device memory uses it). For callers that build
 * once per plan -- the C++ drop-in (include/taps_b200/aux_graph_b200.hpp).
 * The scratch memory stays allocated for the thread, sized by its largest
 * build so far. */
tp_status tp_plan_execute_host_scratch(tp_plan* plan, const tp_build_opts* opts,
                                       tp_aux_index* index_out, tp_cost_tensors* host_out);
/* tp_build_cost_tensors_multi on an analysed plan: per-device copies of the
 * plan (arenas, uploads) are kept on it for repeated executes. */
tp_status tp_plan_execute_host_multi(tp_plan* plan, const int32_t* devices, int32_t num_devices,
                                     tp_aux_index* index_out, tp_cost_tensors* host_out);
/* Re-price an analysed plan under other intra/inter bandwidths (a sweep over
 * the intra/inter ratio, cfg3): nothing of the host analysis depends on them,
 * so the next execute uploads the new pricing tables and rebuilds. Results
 * equal a fresh build with ClusterTopology{node_count, local_device_num,
 * intra_bandwidth, inter_bandwidth, device_memory} (graph.hpp:189-199). */
tp_status tp_plan_set_bandwidth(tp_plan* plan, double intra_bandwidth, double inter_bandwidth);
/* Synchronise the plan's stream and turn a kernel-flagged error into a
 * status (and tp_last_error message). */
tp_status tp_plan_check_errors(tp_plan* plan);
/* Number of kernel launches the last execute issued. */
int64_t tp_plan_last_launches(const tp_plan* plan);
/* Optional cudaEvent_t pair recorded on the launch stream immediately before
 * and after the fused kernel of every execute; NULL disables. */
tp_status tp_plan_set_profile_events(tp_plan* plan, void* start_event, void* stop_event);
/* Diagnostics: when on, execute records device timestamps of its phases.
 * tp_plan_timeline (synchronous) returns, in ns after the kernel's first block
 * started: node rows done, first class pair done, all pairs done, first
 * fan-out tile past its wait, kernel end (-1 where a phase did not run). */
tp_status tp_plan_set_timeline(tp_plan* plan, int32_t on);
tp_status tp_plan_timeline(tp_plan* plan, int64_t ns_out[5]);
/* Per-item trace of the last execute with the timeline on (uint32 values).
 * section 0: class pairs (start, duration, edge class); 1: node-class rows
 * (start, duration); 2: fan-out ranges (start, wait for inputs, duration) --
 * times in ns, starts after the kernel's first CTA started; 3: per class
 * pair (warp form), SM clocks of the pricing sections (closure, axes,
 * inference), inferred ops, unified axes, unified device dims, closure
 * rounds, 0; 4: per warp of the launch, when it left the pricing phase (ns).
 * out == NULL returns the entry count in *count; else *count must equal it
 * and out holds 3, 2, 3, 8 or 1 values per entry. */
tp_status tp_plan_timeline_detail(tp_plan* plan, int32_t section, uint32_t* out, int64_t* count);

/* --- batches of independent scenarios (cfg5 sweeps) ------------------------
 * A sweep of (model, mesh, bandwidth-ratio) scenarios is a set of independent
 * build_auxiliary_graph calls (aux_graph.hpp:211; the reference's CLI/tests
 * loop over them one at a time, pipeline.hpp:152-168 per scenario). The
 * batch entry points run the host analysis of many scenarios on a pool of
 * host threads and keep the device busy with one stream per worker, so the
 * per-build latencies (analysis, descriptor copy, launch, D2H) overlap.
 *
 * tp_plan_create_batch: plans_out[i] / status_out[i] for scenario i (a failed
 * analysis leaves plans_out[i] = NULL and its tp_status in status_out[i]).
 * host_threads <= 0 picks the hardware concurrency (capped at 32).
 * Returns TP_OK when every scenario succeeded, else the status of the first
 * failing one (its message in tp_last_error). */
tp_status tp_plan_create_batch(const tp_graph_desc* const* graphs,
                               const tp_topology_desc* const* topos, int32_t n,
                               int32_t device, int32_t host_threads,
                               tp_plan** plans_out, int32_t* status_out);
/* Execute plans[i] into HOST pointers host_outs[i] (like tp_plan_execute_host,
 * whole graphs, nodes included; every tp_cost_tensors field is honoured).
 * Plans on one device whose outputs are only the six SoA tensors run as ONE
 * batched launch (tp_plan_execute_batch) with one D2H per tensor kind; AuxEdge
 * records or solver minima, or plans on several devices, take one
 * tp_plan_execute_host per plan on the worker threads. index_outs may be NULL. Plans with their own
 * uploaded arena (tp_plan_upload called) keep it; the others borrow a pooled
 * per-worker arena for the duration of the call. NULL plans are skipped with
 * status TP_ERR_INVALID_ARGUMENT. */
tp_status tp_plan_execute_host_batch(tp_plan* const* plans, int32_t n,
                                     tp_aux_index* index_outs,
                                     tp_cost_tensors* host_outs,
                                     int32_t host_threads, int32_t* status_out);

/* The one-shot sweep: build_auxiliary_graph of every (graphs[i], topos[i])
 * into HOST pointers host_outs[i] (the six SoA tensors; index_outs optional),
 * equal to n calls of tp_build_cost_tensors. Pipelined in chunks of
 * scenarios: the host analysis of chunk k + 1 (host_threads workers) runs
 * while the device builds chunk k, and when the caller's slices of a tensor
 * kind are contiguous pinned memory the kernels write them directly (no
 * staging, no separate D2H), so the host link streams for the whole call.
 * Returns TP_OK when every scenario succeeded, else the first failing one's
 * status; status_out[i] per scenario. */
tp_status tp_build_cost_tensors_batch(const tp_graph_desc* const* graphs,
                                      const tp_topology_desc* const* topos, int32_t n,
                                      int32_t device, int32_t host_threads,
                                      tp_aux_index* index_outs, tp_cost_tensors* host_outs,
                                      int32_t* status_out);

/* Build every plan into DEVICE pointers device_outs[i] with ONE persistent
 * launch on `stream` (NULL = plans[0]'s stream): the units and output ranges
 * of all plans form one work queue, so the latency-bound pricing of many small
 * scenarios overlaps instead of paying one launch each. Every plan's results
 * equal tp_plan_execute's (whole graphs). Plans must live on one device;
 * a plan not yet uploaded is uploaded on `stream` (a plan uploaded on another
 * stream must have completed that upload). Errors are per plan:
 * tp_plan_check_errors(plans[i]). */
tp_status tp_plan_execute_batch(tp_plan* const* plans, int32_t n,
                                tp_cost_tensors* device_outs, void* stream);
/* Kernel launches of the last batched execute on `device` (the inference
 * pass and the build launches of all its plans together). */
int64_t tp_batch_last_launches(int32_t device);
/* Optional cudaEvent_t pair recorded on the launch stream of every batched
 * execute on `device`, immediately before its first kernel (the inference
 * pass) and after its last (the launches are enqueued back to back, so the
 * pair times the batch's device work without the host's preparation); NULL
 * disables. */
tp_status tp_batch_set_profile_events(int32_t device, void* start_event, void* stop_event);

/* price_assignment (aux_graph.hpp:326-348) of k strategy assignments on the
 * device, both cost modes at once: assignments [k * num_ops] (the strategy
 * index of every operator, DEVICE memory), t = the plan's six DEVICE cost
 * tensors from tp_plan_execute; out (DEVICE, [k], any may be NULL): the
 * topology-mode cost (sum of cost_s), the volume-mode cost (sum of
 * volume_bytes) and the memory sum, each accumulated in the reference's
 * order. Asynchronous on `stream`. Used for the TAPS-vs-volume ratio of a
 * sweep (pipeline.hpp:152-168: both winners priced in topology mode). */
tp_status tp_plan_price_assignments(tp_plan* plan, const tp_cost_tensors* t,
                                    const int32_t* assignments, int32_t k,
                                    double* cost_s, double* volume_bytes,
                                    double* memory_bytes, void* stream);

/* The reference's ILP of this build as CPLEX LP text, written to `path`:
 * byte-identical to topoplan::export_lp(topoplan::formulate(aux, mode,
 * device_memory)) (solver.hpp:69-176, 578-600; mode_volume selects
 * CostMode::kVolume), produced straight from the plan's index and the six HOST
 * cost tensors of tp_plan_execute_host (include/taps_b200/lp_export.hpp),
 * without materialising the problem. *bytes_out (optional) = bytes written. */
tp_status tp_plan_export_lp(const tp_plan* plan, const tp_cost_tensors* host_tensors, int32_t mode_volume,
                            double device_memory, const char* path, int64_t* bytes_out);

/* Strategy table of an operator with p axes on N devices, in the reference's
 * enumeration order (layout.hpp:270-328), produced on the device.
 * degrees[S*p], device_map[S*p], matrix_dims[S*p] (outermost first, padded
 * with 0 after the canonical depth), matrix_depth[S]. Returns S via *count.
 * Pass NULL arrays to query the count only. */
tp_status tp_enumerate_strategies(int32_t p, int64_t total_devices,
                                  int64_t* count, int64_t* degrees,
                                  int32_t* device_map, int64_t* matrix_dims,
                                  int32_t* matrix_depth);

/* Verification export of one redistribution (redistribution.hpp:557-561 +
 * cost_model.hpp:233-263), evaluated by the device kernel's code path on the
 * GPU. Layout matrices outermost-first as DeviceMatrix::dims. Outputs: the
 * unified matrix (outermost first), unified from/to maps, the op list as
 * (kind, device_dim, tensor_axis, dest_axis, fallback) int32 quintuples, the
 * per-op ct and seconds, and the plan volume/seconds for tensor_bytes. */
typedef struct tp_redist_query {
  int32_t rank;
  const int64_t* shape;
  int32_t from_depth; const int64_t* from_dims; const int32_t* from_map;
  int32_t to_depth;   const int64_t* to_dims;   const int32_t* to_map;
  double tensor_bytes;
  int32_t local_device_num;
  double intra_bandwidth;
  double inter_bandwidth;
} tp_redist_query;

#define TP_MAX_UNIFIED_DEPTH 16
#define TP_MAX_UNIFIED_RANK 32
#define TP_MAX_PLAN_OPS 64

typedef struct tp_redist_result {
  int32_t status;       /* tp_error_kind; 0 = ok */
  int32_t depth;
  int64_t dims[TP_MAX_UNIFIED_DEPTH];
  int32_t urank;
  int64_t shape[TP_MAX_UNIFIED_RANK];
  int32_t from_map[TP_MAX_UNIFIED_RANK];
  int32_t to_map[TP_MAX_UNIFIED_RANK];
  int32_t num_ops;
  int32_t ops[TP_MAX_PLAN_OPS][5];
  int64_t op_ct[TP_MAX_PLAN_OPS];
  double op_seconds[TP_MAX_PLAN_OPS];
  double volume_bytes;
  double seconds;
} tp_redist_result;

tp_status tp_redistribute_batch(const tp_redist_query* queries, int32_t n,
                                tp_redist_result* results);
/* Same, choosing the kernel form of the pair path: 1 = warp per pair (used
 * for small class tables), 2 = thread per pair (large ones). */
tp_status tp_redistribute_batch_form(const tp_redist_query* queries, int32_t n,
                                     tp_redist_result* results, int32_t form);
/* Force the pair form of a plan: 0 = by size (default), 1 = warp, 2 = thread. */
tp_status tp_plan_set_pair_form(tp_plan* plan, int32_t form);

const char* tp_last_error(void);
int32_t tp_last_error_kind(void);
int32_t tp_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TAPS_B200_H_ */
