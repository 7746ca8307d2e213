/*
 * taps_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference's cost-tensor build
 * (topoplan::build_auxiliary_graph, /root/reference/proj/include/topoplan/
 * aux_graph.hpp:211-315, and everything it calls). It is the parity checker
 * for the CUDA engine: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it. The product path never calls it.
 *
 * Parity of this restatement is pinned against (1) the reference's own
 * golden vectors (tests/golden/, from the GTest suites) and (2) the
 * reference itself compiled from /root/reference (oracle/_ref, see
 * oracle/Makefile), on seeded random graphs.
 *
 * It shares only the *data types* of include/taps_b200.h (descriptor and
 * output structs) with the engine, none of its code.
 */
#ifndef TAPS_ORACLE_H_
#define TAPS_ORACLE_H_

#include "../include/taps_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Sizes of the auxiliary graph the build would produce (no pricing). */
int oracle_sizes(const tp_graph_desc* g, const tp_topology_desc* t,
                 int64_t* num_aux_nodes, int64_t* num_aux_edges,
                 int64_t* num_rows);

/* Full build with the reference's memo semantics (first writer per
 * (shape, from-layout, to-layout) key, aux_graph.hpp:257-271).
 * Returns tp_status; *error_kind receives the tp_error_kind. */
int oracle_build(const tp_graph_desc* g, const tp_topology_desc* t,
                 tp_aux_index* index, tp_cost_tensors* out,
                 int32_t* error_kind);

/* Un-memoised build: every pair priced with its own edge's tensor bytes,
 * i.e. topoplan::edge_weight (aux_graph.hpp:184-207) for every aux edge. */
int oracle_build_unmemoized(const tp_graph_desc* g, const tp_topology_desc* t,
                            tp_aux_index* index, tp_cost_tensors* out,
                            int32_t* error_kind);

/* One redistribution + its pricing (redistribution.hpp:557-561,
 * 533-553; cost_model.hpp:176-263). Returns tp_error_kind (0 = ok). */
int oracle_redistribute(const tp_redist_query* q, tp_redist_result* r);

/* Strategy table (layout.hpp:222-328). Returns the count, or -1 on error;
 * arrays may be NULL. matrix_dims outermost first, padded with 0 to p. */
int64_t oracle_enumerate(int32_t p, int64_t total_devices, int64_t* degrees,
                         int32_t* device_map, int64_t* matrix_dims,
                         int32_t* matrix_depth);
int64_t oracle_strategy_count(int32_t p, int64_t total_devices);

/* ct of an AllReduce / AllGather group (cost_model.hpp:75-135);
 * matrix dims outermost first. */
int64_t oracle_ct_allreduce(int32_t depth, const int64_t* dims, int32_t rank,
                            const int32_t* map, int64_t local_device_num);
void oracle_ct_allgather_dim(int32_t depth, const int64_t* dims, int32_t rank,
                             const int32_t* map, int32_t gather_dim,
                             int64_t local_device_num, int64_t* ct,
                             int64_t* repeat_num, int64_t* group_in_node);

#ifdef __cplusplus
}
#endif

#endif /* TAPS_ORACLE_H_ */
