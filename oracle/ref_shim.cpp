// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/topoplan/*.hpp), compiled by oracle/Makefile
// into oracle/_ref/libtopoplan_ref.so. It lets the Python tests and bench.py
// run the reference's own build_auxiliary_graph / redistribute / solve on the
// same flattened descriptors the CUDA engine consumes:
//   - to pin the C restatement (oracle/taps_oracle.c) against the reference,
//   - to generate the golden fixtures under tests/golden/,
//   - as the timed CPU baseline ("kind": "reference") in bench.py.
// No reference source is copied here; the headers are included from their
// read-only location at build time only.

#include <atomic>
#include <chrono>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "topoplan/aux_graph.hpp"
#include "topoplan/models.hpp"
#include "topoplan/solver.hpp"

#include "../include/taps_b200.h"
#include "../include/taps_b200/models_b200.hpp"  // the C++ composer, checked against models.py

using namespace topoplan;

namespace {

// POD thread-locals only: a non-trivial thread_local in a dlopen'ed library
// crashed when numpy's runtime was loaded first.
thread_local char g_last_msg[1024];

void set_msg(const char* m) {
  std::strncpy(g_last_msg, m, sizeof(g_last_msg) - 1);
  g_last_msg[sizeof(g_last_msg) - 1] = 0;
}

std::string op_name(int id) { return "op" + std::to_string(id); }
std::string t_name(int id) { return "t" + std::to_string(id); }

ComputationGraph to_graph(const tp_graph_desc* g) {
  ComputationGraph graph;
  for (int i = 0; i < g->num_ops; ++i) {
    OperatorNode op;
    op.id = op_name(g->op_id[i]);
    op.kind = OpKind::kOther;
    const int t0 = g->op_tensor_begin[i], t1 = g->op_tensor_begin[i + 1];
    for (int t = t0; t < t1; ++t) {
      TensorSpec spec;
      spec.name = t_name(g->tensor_name[t]);
      spec.shape.assign(g->shape + g->tensor_shape_begin[t],
                        g->shape + g->tensor_shape_begin[t + 1]);
      spec.element_size = g->tensor_element_size[t];
      if (t - t0 < g->op_num_inputs[i]) op.inputs.push_back(spec);
      else op.outputs.push_back(spec);
    }
    for (int a = g->op_axis_begin[i]; a < g->op_axis_begin[i + 1]; ++a) {
      OperatorAxis axis;
      axis.name = "a" + std::to_string(a - g->op_axis_begin[i]);
      for (int s = g->axis_slice_begin[a]; s < g->axis_slice_begin[a + 1]; ++s) {
        axis.slices.push_back({t_name(g->slice_tensor[s]), g->slice_dim[s]});
      }
      op.axes.push_back(axis);
    }
    graph.operators.push_back(op);
  }
  for (int e = 0; e < g->num_edges; ++e) {
    graph.edges.push_back({op_name(g->edge_from[e]), op_name(g->edge_to[e]),
                           t_name(g->edge_tensor[e])});
  }
  return graph;
}

ClusterTopology to_topo(const tp_topology_desc* t) {
  ClusterTopology topo;
  topo.node_count = t->node_count;
  topo.local_device_num = t->local_device_num;
  topo.intra_bandwidth = t->intra_bandwidth;
  topo.inter_bandwidth = t->inter_bandwidth;
  topo.device_memory = t->device_memory;
  return topo;
}

void export_aux(const AuxiliaryGraph& aux, tp_aux_index* index,
                tp_cost_tensors* out) {
  const int n_ops = static_cast<int>(aux.graph.operators.size());
  if (index) {
    if (index->node_base) {
      for (int i = 0; i < n_ops; ++i)
        index->node_base[i] = aux.nodes_of_op[i].empty() ? 0 : aux.nodes_of_op[i][0];
      index->node_base[n_ops] = static_cast<int64_t>(aux.nodes.size());
    }
    if (index->edge_base) {
      for (std::size_t e = 0; e < aux.edge_base.size(); ++e) index->edge_base[e] = aux.edge_base[e];
      index->edge_base[aux.edge_base.size()] = static_cast<int64_t>(aux.edges.size());
    }
    for (std::size_t e = 0; e < aux.graph.edges.size(); ++e) {
      if (index->edge_from_op) index->edge_from_op[e] = aux.graph.find_op(aux.graph.edges[e].from);
      if (index->edge_to_op) index->edge_to_op[e] = aux.graph.find_op(aux.graph.edges[e].to);
    }
    for (int i = 0; i < n_ops; ++i) {
      if (index->in_degree) index->in_degree[i] = aux.in_degree_of[i];
      if (index->out_degree) index->out_degree[i] = aux.out_degree_of[i];
      if (index->topo_order) index->topo_order[i] = aux.topo_order[i];
    }
  }
  if (!out) return;
  for (std::size_t n = 0; n < aux.nodes.size(); ++n) {
    if (out->node_intra_cost_s) out->node_intra_cost_s[n] = aux.nodes[n].intra_cost_s;
    if (out->node_intra_volume_bytes) out->node_intra_volume_bytes[n] = aux.nodes[n].intra_volume_bytes;
    if (out->node_memory_bytes) out->node_memory_bytes[n] = aux.nodes[n].memory_bytes;
  }
  for (std::size_t e = 0; e < aux.edges.size(); ++e) {
    const AuxEdge& ae = aux.edges[e];
    if (out->edge_cost_s) out->edge_cost_s[e] = ae.cost_s;
    if (out->edge_volume_bytes) out->edge_volume_bytes[e] = ae.volume_bytes;
    if (out->edge_memory_bytes) out->edge_memory_bytes[e] = ae.memory_bytes;
    if (out->aux_edge_records) {
      static_assert(sizeof(AuxEdge) == 40, "AuxEdge layout");
      std::memcpy(static_cast<char*>(out->aux_edge_records) + e * 40, &ae, 40);
    }
  }
  // cond_min of solver.hpp:239-253, both modes
  std::int64_t row = 0;
  for (std::size_t e = 0; e < aux.graph.edges.size(); ++e) {
    const int u = aux.graph.find_op(aux.graph.edges[e].from);
    const int w = aux.graph.find_op(aux.graph.edges[e].to);
    const int su_n = aux.strategies_of(u), sw_n = aux.strategies_of(w);
    for (int su = 0; su < su_n; ++su, ++row) {
      double mc = std::numeric_limits<double>::infinity();
      double mv = std::numeric_limits<double>::infinity();
      for (int sw = 0; sw < sw_n; ++sw) {
        const AuxEdge& ae = aux.edges[aux.edge_base[e] + su * sw_n + sw];
        mc = std::min(mc, ae.cost_s);
        mv = std::min(mv, ae.volume_bytes);
      }
      if (out->row_min_cost_s) out->row_min_cost_s[row] = mc;
      if (out->row_min_volume_bytes) out->row_min_volume_bytes[row] = mv;
    }
  }
  // pair_min straight from the reference solver's own make_context (solver.hpp:218-287)
  if (out->edge_pair_min_cost_s || out->edge_pair_min_volume_bytes) {
    const detail::SearchContext ct = detail::make_context(aux, CostMode::kTopology, 0.0);
    const detail::SearchContext cv = detail::make_context(aux, CostMode::kVolume, 0.0);
    for (std::size_t e = 0; e < aux.graph.edges.size(); ++e) {
      if (out->edge_pair_min_cost_s) out->edge_pair_min_cost_s[e] = ct.pair_min[e];
      if (out->edge_pair_min_volume_bytes) out->edge_pair_min_volume_bytes[e] = cv.pair_min[e];
    }
  }
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    set_msg("");
    return TP_OK;
  } catch (const Error& e) {
    set_msg(e.what());
    return TP_ERR_TOPOPLAN;
  } catch (const std::out_of_range& e) {
    set_msg(e.what());
    return TP_ERR_OUT_OF_RANGE;
  } catch (const std::exception& e) {
    set_msg(e.what());
    return TP_ERR_INVALID_ARGUMENT;
  }
}

void dump_graph(std::ostringstream& o, const ComputationGraph& g) {
  // tiny JSON writer (the reference's io.hpp needs the absent json.hpp)
  o << "{\"operators\":[";
  for (std::size_t i = 0; i < g.operators.size(); ++i) {
    const OperatorNode& op = g.operators[i];
    if (i) o << ",";
    o << "{\"id\":\"" << op.id << "\",\"kind\":\"" << to_string(op.kind) << "\",";
    auto tensors = [&](const char* key, const std::vector<TensorSpec>& ts) {
      o << "\"" << key << "\":[";
      for (std::size_t t = 0; t < ts.size(); ++t) {
        if (t) o << ",";
        o << "{\"name\":\"" << ts[t].name << "\",\"shape\":[";
        for (std::size_t d = 0; d < ts[t].shape.size(); ++d) o << (d ? "," : "") << ts[t].shape[d];
        o << "],\"element_size\":" << ts[t].element_size << "}";
      }
      o << "],";
    };
    tensors("inputs", op.inputs);
    tensors("outputs", op.outputs);
    o << "\"axes\":[";
    for (std::size_t a = 0; a < op.axes.size(); ++a) {
      if (a) o << ",";
      o << "{\"name\":\"" << op.axes[a].name << "\",\"slices\":[";
      for (std::size_t s = 0; s < op.axes[a].slices.size(); ++s) {
        if (s) o << ",";
        o << "{\"tensor\":\"" << op.axes[a].slices[s].tensor << "\",\"dim\":" << op.axes[a].slices[s].dim << "}";
      }
      o << "]}";
    }
    o << "]}";
  }
  o << "],\"edges\":[";
  for (std::size_t e = 0; e < g.edges.size(); ++e) {
    if (e) o << ",";
    o << "{\"from\":\"" << g.edges[e].from << "\",\"to\":\"" << g.edges[e].to
      << "\",\"tensor\":\"" << g.edges[e].tensor << "\"}";
  }
  o << "]}";
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_msg; }

// build_auxiliary_graph (aux_graph.hpp:211) -> SoA / AoS export.
int ref_build(const tp_graph_desc* g, const tp_topology_desc* t,
              tp_aux_index* index, tp_cost_tensors* out) {
  return guarded([&] {
    const AuxiliaryGraph aux = build_auxiliary_graph(to_graph(g), to_topo(t));
    export_aux(aux, index, out);
  });
}

// edge_weight (aux_graph.hpp:184) for every aux edge: the un-memoised path.
int ref_build_unmemoized(const tp_graph_desc* g, const tp_topology_desc* t,
                         tp_cost_tensors* out) {
  return guarded([&] {
    const AuxiliaryGraph aux = build_auxiliary_graph(to_graph(g), to_topo(t));
    for (std::size_t e = 0; e < aux.graph.edges.size(); ++e) {
      const int u = aux.graph.find_op(aux.graph.edges[e].from);
      const int w = aux.graph.find_op(aux.graph.edges[e].to);
      for (int su = 0; su < aux.strategies_of(u); ++su) {
        for (int sw = 0; sw < aux.strategies_of(w); ++sw) {
          const EdgeWeight wt = edge_weight(aux.graph, static_cast<int>(e),
                                            aux.nodes[aux.nodes_of_op[u][su]],
                                            aux.nodes[aux.nodes_of_op[w][sw]], aux.topo);
          const int id = aux.edge_id(static_cast<int>(e), su, sw);
          if (out->edge_cost_s) out->edge_cost_s[id] = wt.cost_s;
          if (out->edge_volume_bytes) out->edge_volume_bytes[id] = wt.volume_bytes;
          if (out->edge_memory_bytes) out->edge_memory_bytes[id] = wt.memory_bytes;
        }
      }
    }
  });
}

// Wall time of `iters` builds on each of `threads` threads (pure function of
// immutable inputs, so concurrent builds are safe).
int ref_bench_build(const tp_graph_desc* g, const tp_topology_desc* t,
                    int iters, int threads, double* seconds, int64_t* aux_edges) {
  return guarded([&] {
    const ComputationGraph graph = to_graph(g);
    const ClusterTopology topo = to_topo(t);
    std::vector<std::int64_t> counts(threads, 0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int th = 0; th < threads; ++th) {
      pool.emplace_back([&, th] {
        for (int i = 0; i < iters; ++i) {
          const AuxiliaryGraph aux = build_auxiliary_graph(graph, topo);
          counts[th] += static_cast<std::int64_t>(aux.edges.size());
        }
      });
    }
    for (auto& th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    std::int64_t total = 0;
    for (auto c : counts) total += c;
    *aux_edges = total;
  });
}

// A sweep of independent scenarios on a pool of `threads` host threads, each
// scenario one unmodified build_auxiliary_graph call (the reference has no
// intra-build parallelism; scenarios are pure functions).
int ref_bench_sweep(const tp_graph_desc* const* g, const tp_topology_desc* const* t, int n, int threads,
                    double* seconds, int64_t* aux_edges) {
  return guarded([&] {
    std::vector<ComputationGraph> graphs;
    std::vector<ClusterTopology> topos;
    for (int i = 0; i < n; ++i) {
      graphs.push_back(to_graph(g[i]));
      topos.push_back(to_topo(t[i]));
    }
    std::vector<std::int64_t> counts(threads, 0);
    std::atomic<int> next{0};
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int th = 0; th < threads; ++th) {
      pool.emplace_back([&, th] {
        for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) {
          const AuxiliaryGraph aux = build_auxiliary_graph(graphs[i], topos[i]);
          counts[th] += static_cast<std::int64_t>(aux.edges.size());
        }
      });
    }
    for (auto& th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    std::int64_t total = 0;
    for (auto c : counts) total += c;
    *aux_edges = total;
  });
}

// redistribute + plan_volume + redistribution_cost, with per-op ct from
// collective_cost_detail (redistribution.hpp:557; cost_model.hpp:176-263).
int ref_redistribute(const tp_redist_query* q, tp_redist_result* r) {
  std::memset(r, 0, sizeof(*r));
  return guarded([&] {
    TensorLayout from, to;
    from.spec = {"t", std::vector<std::int64_t>(q->shape, q->shape + q->rank), 4};
    to.spec = from.spec;
    from.matrix = DeviceMatrix(std::vector<std::int64_t>(q->from_dims, q->from_dims + q->from_depth));
    to.matrix = DeviceMatrix(std::vector<std::int64_t>(q->to_dims, q->to_dims + q->to_depth));
    from.map = TensorMap(std::vector<int>(q->from_map, q->from_map + q->rank));
    to.map = TensorMap(std::vector<int>(q->to_map, q->to_map + q->rank));
    const RedistPlan plan = redistribute(from, to);
    if (plan.matrix.depth() > TP_MAX_UNIFIED_DEPTH || static_cast<int>(plan.shape.size()) > TP_MAX_UNIFIED_RANK ||
        static_cast<int>(plan.ops.size()) > TP_MAX_PLAN_OPS) {
      throw std::runtime_error("capacity");
    }
    r->depth = plan.matrix.depth();
    for (int k = 0; k < r->depth; ++k) r->dims[k] = plan.matrix.dims[k];
    r->urank = static_cast<int>(plan.shape.size());
    for (int i = 0; i < r->urank; ++i) {
      r->shape[i] = plan.shape[i];
      r->from_map[i] = plan.from_map[i];
      r->to_map[i] = plan.to_map[i];
    }
    r->num_ops = static_cast<int>(plan.ops.size());
    const BandwidthEnv env{q->intra_bandwidth, q->inter_bandwidth, q->local_device_num};
    TensorMap working = plan.from_map;
    for (int i = 0; i < r->num_ops; ++i) {
      const RedistOp& op = plan.ops[i];
      r->ops[i][0] = static_cast<int>(op.kind);
      r->ops[i][1] = op.device_dim;
      r->ops[i][2] = op.tensor_axis;
      r->ops[i][3] = op.dest_axis;
      r->ops[i][4] = op.fallback ? 1 : 0;
      const double shard = shard_bytes_under(plan.matrix, working, q->tensor_bytes);
      if (op.kind != RedistOpKind::kSlice) {
        CollectiveCall call{op.kind == RedistOpKind::kAllGather ? CollectiveKind::kAllGather
                                                                : CollectiveKind::kAllToAll,
                            plan.matrix.extent(op.device_dim), shard, plan.matrix, working,
                            op.device_dim};
        const CollectiveCost c = collective_cost_detail(call, env);
        r->op_ct[i] = c.ct;
        r->op_seconds[i] = c.seconds;
      }
      switch (op.kind) {
        case RedistOpKind::kSlice: working.entries[op.tensor_axis] = op.device_dim; break;
        case RedistOpKind::kAllGather: working.entries[op.tensor_axis] = -1; break;
        case RedistOpKind::kAllToAll:
          working.entries[op.tensor_axis] = -1;
          working.entries[op.dest_axis] = op.device_dim;
          break;
      }
    }
    r->volume_bytes = plan_volume(plan, q->tensor_bytes);
    r->seconds = redistribution_cost(plan, q->tensor_bytes, env);
  });
}

// enumerate_strategies (layout.hpp:270-328).
int64_t ref_enumerate(int32_t p, int64_t total, int64_t* degrees, int32_t* device_map,
                      int64_t* matrix_dims, int32_t* matrix_depth) {
  std::int64_t n = -1;
  int st = guarded([&] {
    OperatorNode op;
    op.id = "probe";
    op.inputs = {{"t", std::vector<std::int64_t>(p, 64), 4}};
    for (int a = 0; a < p; ++a) op.axes.push_back({"a" + std::to_string(a), {{"t", a}}});
    const auto s = enumerate_strategies(op, total);
    n = static_cast<std::int64_t>(s.size());
    for (std::int64_t i = 0; i < n; ++i) {
      for (int a = 0; a < p; ++a) {
        if (degrees) degrees[i * p + a] = s[i].degrees[a];
        if (device_map) device_map[i * p + a] = s[i].device_map[a];
        if (matrix_dims)
          matrix_dims[i * p + a] = a < s[i].device_matrix.depth() ? s[i].device_matrix.dims[a] : 0;
      }
      if (matrix_depth) matrix_depth[i] = s[i].device_matrix.depth();
    }
  });
  return st == TP_OK ? n : -1;
}

int64_t ref_strategy_count(int32_t p, int64_t total) {
  std::int64_t n = -1;
  int st = guarded([&] { n = strategy_count(p, total); });
  return st == TP_OK ? n : -1;
}

int64_t ref_ct_allreduce(int32_t depth, const int64_t* dims, int32_t rank,
                         const int32_t* map, int64_t local) {
  return infer_ct_allreduce(DeviceMatrix(std::vector<std::int64_t>(dims, dims + depth)),
                            TensorMap(std::vector<int>(map, map + rank)), local);
}

void ref_ct_allgather_dim(int32_t depth, const int64_t* dims, int32_t rank,
                          const int32_t* map, int32_t g, int64_t local, int64_t* ct,
                          int64_t* repeat, int64_t* gin) {
  const AllGatherCt r =
      infer_ct_allgather_dim(DeviceMatrix(std::vector<std::int64_t>(dims, dims + depth)),
                             TensorMap(std::vector<int>(map, map + rank)), g, local);
  *ct = r.ct;
  *repeat = r.repeat_num;
  *gin = r.group_in_node;
}

// formulate + solve (solver.hpp:69, 417). When the cost arrays are given,
// they replace the reference-built payloads first, so the reference solver
// runs on externally built (e.g. GPU) cost tensors.
int ref_solve(const tp_graph_desc* g, const tp_topology_desc* t, int mode_volume,
              double memory_bound, int threads, int64_t max_nodes,
              const tp_cost_tensors* given, int32_t* strategy_per_op, double* objective,
              int32_t* feasible, int32_t* optimal, double* root_bound,
              int64_t* nodes_explored) {
  return guarded([&] {
    AuxiliaryGraph aux = build_auxiliary_graph(to_graph(g), to_topo(t));
    if (given) {
      for (std::size_t n = 0; n < aux.nodes.size(); ++n) {
        if (given->node_intra_cost_s) aux.nodes[n].intra_cost_s = given->node_intra_cost_s[n];
        if (given->node_intra_volume_bytes) aux.nodes[n].intra_volume_bytes = given->node_intra_volume_bytes[n];
        if (given->node_memory_bytes) aux.nodes[n].memory_bytes = given->node_memory_bytes[n];
      }
      for (std::size_t e = 0; e < aux.edges.size(); ++e) {
        if (given->edge_cost_s) aux.edges[e].cost_s = given->edge_cost_s[e];
        if (given->edge_volume_bytes) aux.edges[e].volume_bytes = given->edge_volume_bytes[e];
        if (given->edge_memory_bytes) aux.edges[e].memory_bytes = given->edge_memory_bytes[e];
      }
      for (auto& ve : aux.virtual_edges) {
        ve.cost_s = aux.nodes[ve.to_node].intra_cost_s;
        ve.volume_bytes = aux.nodes[ve.to_node].intra_volume_bytes;
        ve.memory_bytes = aux.nodes[ve.to_node].memory_bytes;
      }
    }
    const IlpProblem problem =
        formulate(aux, mode_volume ? CostMode::kVolume : CostMode::kTopology, memory_bound);
    SolveOptions opts;
    opts.threads = threads;
    opts.max_nodes = max_nodes;
    const PlanSolution s = solve(problem, opts);
    *feasible = s.feasible;
    *optimal = s.optimal;
    *objective = s.objective;
    *root_bound = s.root_lower_bound;
    *nodes_explored = s.nodes_explored;
    for (std::size_t i = 0; i < s.strategy_per_op.size(); ++i) strategy_per_op[i] = s.strategy_per_op[i];
  });
}

// price_assignment (aux_graph.hpp:326-348) of k assignments [k * num_ops]
// on the reference's own build: the topology-mode cost, the volume-mode cost
// and the memory sum of each (arrays of length k, any may be NULL).
int ref_price_assignments(const tp_graph_desc* g, const tp_topology_desc* t, const int32_t* asg, int k,
                          double* cost_s, double* volume_bytes, double* memory_bytes) {
  return guarded([&] {
    const AuxiliaryGraph aux = build_auxiliary_graph(to_graph(g), to_topo(t));
    const std::size_t nops = aux.graph.operators.size();
    for (int j = 0; j < k; ++j) {
      const std::vector<int> a(asg + (std::size_t)j * nops, asg + (std::size_t)(j + 1) * nops);
      const AssignmentPrice pt = price_assignment(aux, a, CostMode::kTopology);
      const AssignmentPrice pv = price_assignment(aux, a, CostMode::kVolume);
      if (cost_s) cost_s[j] = pt.cost;
      if (volume_bytes) volume_bytes[j] = pv.cost;
      if (memory_bytes) memory_bytes[j] = pt.memory_bytes;
    }
  });
}

// export_lp (solver.hpp:578) of the reference-built problem; returns the
// length written (or needed).
int64_t ref_export_lp(const tp_graph_desc* g, const tp_topology_desc* t, int mode_volume,
                      double memory_bound, char* buf, int64_t cap) {
  std::string lp;
  int st = guarded([&] {
    const AuxiliaryGraph aux = build_auxiliary_graph(to_graph(g), to_topo(t));
    lp = export_lp(formulate(aux, mode_volume ? CostMode::kVolume : CostMode::kTopology,
                             memory_bound));
  });
  if (st != TP_OK) return -1;
  if (buf && cap > 0) {
    const std::int64_t n = std::min<std::int64_t>(cap - 1, static_cast<std::int64_t>(lp.size()));
    std::memcpy(buf, lp.data(), static_cast<std::size_t>(n));
    buf[n] = 0;
  }
  return static_cast<std::int64_t>(lp.size());
}

// The C++ composer of include/taps_b200/models_b200.hpp as JSON: which = 0
// gpt_chain(a, b, c, d); which = 1 scenario a of scenario_sweep(b) with its
// topology and ratio appended as {"graph": ..., "topo": [...], "family": ...}.
int64_t ref_composer_json(int which, int64_t a, int64_t b, int64_t c, int64_t d, char* buf, int64_t cap) {
  std::string s;
  int st = guarded([&] {
    std::ostringstream o;
    if (which == 0) {
      dump_graph(o, taps_b200::gpt_chain((int)a, b, c, d));
    } else {
      const auto sweep = taps_b200::scenario_sweep((int)b);
      const auto& sc = sweep.at((size_t)a);
      o << "{\"graph\":";
      dump_graph(o, sc.graph);
      char t[256];
      std::snprintf(t, sizeof(t), ",\"topo\":[%d,%d,%.17g,%.17g,%.17g],\"ratio\":%.17g,\"family\":\"%s\"}",
                    sc.topo.node_count, sc.topo.local_device_num, sc.topo.intra_bandwidth, sc.topo.inter_bandwidth,
                    sc.topo.device_memory, sc.ratio, sc.family.c_str());
      o << t;
    }
    s = o.str();
  });
  if (st != TP_OK) return -1;
  if (buf && cap > 0) {
    const std::int64_t n = std::min<std::int64_t>(cap - 1, static_cast<std::int64_t>(s.size()));
    std::memcpy(buf, s.data(), static_cast<std::size_t>(n));
    buf[n] = 0;
  }
  return static_cast<std::int64_t>(s.size());
}

// models.hpp builders (parse_model_spec + build_graph) as JSON, so the
// Python generators can be checked against the reference's.
int64_t ref_model_json(const char* spec, char* buf, int64_t cap) {
  std::string s;
  int st = guarded([&] {
    std::ostringstream o;
    dump_graph(o, build_graph(parse_model_spec(spec)));
    s = o.str();
  });
  if (st != TP_OK) return -1;
  if (buf && cap > 0) {
    const std::int64_t n = std::min<std::int64_t>(cap - 1, static_cast<std::int64_t>(s.size()));
    std::memcpy(buf, s.data(), static_cast<std::size_t>(n));
    buf[n] = 0;
  }
  return static_cast<std::int64_t>(s.size());
}

}  // extern "C"
