// aux_graph_b200.hpp — header-only C++ drop-in for the reference's hot path.
//
//   topoplan::AuxiliaryGraph aux =
//       taps_b200::build_auxiliary_graph_b200(graph, topo, mode);
//
// replaces topoplan::build_auxiliary_graph (aux_graph.hpp:211-315) for code
// that already uses the topoplan headers: same inputs, same AuxiliaryGraph
// (nodes, nodes_of_op, edges, virtual edges, edge_base, degrees, topological
// order; cost tensors bit-identical), so topoplan::formulate / solve /
// price_assignment / export_lp run unchanged on the result. The cost tensors
// are computed by the B200 engine through the C-ABI (include/taps_b200.h);
// the AuxEdge records are written by the device in topoplan::AuxEdge's own
// 40-byte layout and copied straight into AuxiliaryGraph::edges.
//
// Errors mirror the reference: topoplan::Error where it throws Error,
// std::out_of_range where its layouts.at() would throw; CUDA failures (no
// GPU) throw std::runtime_error — there is no CPU fallback.
//
// AuxNode::layouts (a per-node std::map the solver never reads) is filled
// only when `with_layouts` is set, by tensor_layouts_b200 below.
#ifndef TAPS_B200_AUX_GRAPH_B200_HPP_
#define TAPS_B200_AUX_GRAPH_B200_HPP_

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "topoplan/aux_graph.hpp"
#include "../taps_b200.h"

namespace taps_b200 {

namespace detail {

// Interned, CSR-flattened topoplan::ComputationGraph (tp_graph_desc).
struct FlatGraph {
  std::vector<int32_t> op_id, op_tensor_begin{0}, op_num_inputs, op_axis_begin{0}, tensor_name,
      tensor_shape_begin{0}, tensor_element_size, axis_slice_begin{0}, slice_tensor, slice_dim, edge_from,
      edge_to, edge_tensor;
  std::vector<int64_t> shape;
  tp_graph_desc desc{};

  explicit FlatGraph(const topoplan::ComputationGraph& g) {
    std::unordered_map<std::string, int32_t> ops, names;
    auto oid = [&](const std::string& s) { return ops.emplace(s, (int32_t)ops.size()).first->second; };
    auto nid = [&](const std::string& s) { return names.emplace(s, (int32_t)names.size()).first->second; };
    for (const auto& op : g.operators) {
      op_id.push_back(oid(op.id));
      auto add = [&](const topoplan::TensorSpec& t) {
        tensor_name.push_back(nid(t.name));
        shape.insert(shape.end(), t.shape.begin(), t.shape.end());
        tensor_shape_begin.push_back((int32_t)shape.size());
        tensor_element_size.push_back(t.element_size);
      };
      for (const auto& t : op.inputs) add(t);
      for (const auto& t : op.outputs) add(t);
      op_tensor_begin.push_back((int32_t)tensor_name.size());
      op_num_inputs.push_back((int32_t)op.inputs.size());
      for (const auto& ax : op.axes) {
        for (const auto& s : ax.slices) {
          slice_tensor.push_back(nid(s.tensor));
          slice_dim.push_back(s.dim);
        }
        axis_slice_begin.push_back((int32_t)slice_tensor.size());
      }
      op_axis_begin.push_back((int32_t)axis_slice_begin.size() - 1);
    }
    for (const auto& e : g.edges) {
      edge_from.push_back(oid(e.from));
      edge_to.push_back(oid(e.to));
      edge_tensor.push_back(nid(e.tensor));
    }
    desc.num_ops = (int32_t)g.operators.size();
    desc.op_id = op_id.data();
    desc.op_tensor_begin = op_tensor_begin.data();
    desc.op_num_inputs = op_num_inputs.data();
    desc.op_axis_begin = op_axis_begin.data();
    desc.tensor_name = tensor_name.data();
    desc.tensor_shape_begin = tensor_shape_begin.data();
    desc.shape = shape.data();
    desc.tensor_element_size = tensor_element_size.data();
    desc.axis_slice_begin = axis_slice_begin.data();
    desc.slice_tensor = slice_tensor.data();
    desc.slice_dim = slice_dim.data();
    desc.num_edges = (int32_t)g.edges.size();
    desc.edge_from = edge_from.data();
    desc.edge_to = edge_to.data();
    desc.edge_tensor = edge_tensor.data();
  }
};

[[noreturn]] inline void throw_status(tp_status st) {
  const std::string msg = tp_last_error();
  if (st == TP_ERR_TOPOPLAN) throw topoplan::Error(msg);
  if (st == TP_ERR_OUT_OF_RANGE) throw std::out_of_range(msg);
  throw std::runtime_error("taps_b200: " + msg);
}

inline void check(tp_status st) {
  if (st != TP_OK) throw_status(st);
}

// The structs of include/taps_b200.h this header was compiled with must be
// the library's (tp_cost_tensors grew in ABI 2): refuse another version.
inline void check_abi() {
  if (tp_abi_version() != TP_ABI_VERSION)
    throw std::runtime_error("taps_b200: libtaps_b200 ABI version " + std::to_string(tp_abi_version()) +
                             " differs from the header's " + std::to_string(TP_ABI_VERSION));
}

// TAPS_B200_PROFILE=1: the phases of build_auxiliary_graph_b200 on stderr.
struct PhaseClock {
  bool on = std::getenv("TAPS_B200_PROFILE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  std::string line;
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    char buf[96];
    std::snprintf(buf, sizeof(buf), "%s%s %.2f ms", line.empty() ? "" : ", ", what,
                  std::chrono::duration<double, std::milli>(now - t).count());
    line += buf;
    t = now;
  }
  void report() const {
    if (on) std::fprintf(stderr, "[taps_b200] build_auxiliary_graph_b200: %s\n", line.c_str());
  }
};

// fn(i) for i in [0, n) on up to hardware_concurrency threads (or
// TAPS_B200_THREADS), at least `per_thread` items each (fewer items: the
// calling thread alone); the first exception of any item is rethrown here.
template <typename F>
inline void parallel_for(int n, int per_thread, F&& fn) {
  const char* env = std::getenv("TAPS_B200_THREADS");
  const int hw = env ? std::max(1, std::atoi(env)) : (int)std::max(1u, std::thread::hardware_concurrency());
  const int T = std::min(hw, std::max(1, n / std::max(1, per_thread)));
  if (T <= 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int> next{0};
  std::exception_ptr err;
  std::mutex mu;
  auto run = [&] {
    try {
      for (int i; (i = next.fetch_add(1)) < n;) fn(i);
    } catch (...) {
      std::lock_guard<std::mutex> lk(mu);
      if (!err) err = std::current_exception();
      next.store(n);
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(run);
  run();
  for (auto& x : th) x.join();
  if (err) std::rethrow_exception(err);
}

struct PlanGuard {
  tp_plan* p = nullptr;
  ~PlanGuard() { tp_plan_destroy(p); }
};

}  // namespace detail

// AuxNode::layouts of a strategy (the value layout.hpp:333-370 gives): one
// TensorLayout per tensor NAME -- a name declared twice keeps its last spec --
// over the strategy's device matrix, each tensor dim mapped to the device dim
// of the last axis slicing it (axes in order, slices in order), -1 when none
// does. Called only after a successful build, which has already checked every
// slice's divisibility (the engine's node phase, TP_E_INDIVISIBLE_EXTENT).
inline std::map<std::string, topoplan::TensorLayout> tensor_layouts_b200(const topoplan::OperatorNode& op,
                                                                          const topoplan::OperatorStrategy& st) {
  std::map<std::string, topoplan::TensorLayout> out;
  auto put = [&](const topoplan::TensorSpec& t) {
    topoplan::TensorLayout& l = out[t.name];
    l.spec = t;
    l.matrix = st.device_matrix;
    l.map.entries.assign(t.shape.size(), -1);
  };
  for (const auto& t : op.inputs) put(t);
  for (const auto& t : op.outputs) put(t);
  for (std::size_t a = 0; a < op.axes.size(); ++a)
    for (const auto& sl : op.axes[a].slices) {
      auto it = out.find(sl.tensor);
      if (it != out.end()) it->second.map.entries[sl.dim] = st.device_map[a];
    }
  return out;
}

// Optional side outputs of the build for the solver's search context
// (solver.hpp:218-287): per-(edge, producer strategy) row minima (cond_min,
// rows edge-major) and per-edge minima (pair_min), both cost modes, computed
// on the device; plus find_op of each edge's endpoints. Consumed by
// make_context_b200 (solver_b200.hpp).
struct SolverMinima {
  std::vector<double> row_min_cost_s, row_min_volume_bytes;    // [num_rows]
  std::vector<double> pair_min_cost_s, pair_min_volume_bytes;  // [num_edges]
  std::vector<int32_t> edge_from_op, edge_to_op;               // [num_edges]
};

inline topoplan::AuxiliaryGraph build_auxiliary_graph_b200(const topoplan::ComputationGraph& graph,
                                                           const topoplan::ClusterTopology& topo,
                                                           topoplan::CostMode mode = topoplan::CostMode::kTopology,
                                                           int device = -1, bool with_layouts = false,
                                                           SolverMinima* minima = nullptr) {
  static_assert(sizeof(topoplan::AuxEdge) == 40, "AuxEdge layout differs from the device records");
  detail::check_abi();
  detail::PhaseClock clk;
  topoplan::AuxiliaryGraph aux;
  aux.graph = graph;
  clk.mark("graph copy");
  aux.topo = topo;
  aux.default_mode = mode;

  detail::FlatGraph flat(graph);
  const tp_topology_desc td{topo.node_count, topo.local_device_num, topo.intra_bandwidth, topo.inter_bandwidth,
                            topo.device_memory};
  clk.mark("flatten");
  detail::PlanGuard plan;
  detail::check(tp_plan_create(&flat.desc, &td, device, &plan.p));
  clk.mark("plan create");
  tp_plan_sizes_t sz{};
  detail::check(tp_plan_sizes(plan.p, &sz));
  const int n_ops = (int)graph.operators.size(), n_edges = (int)graph.edges.size();

  std::vector<int64_t> node_base(n_ops + 1), edge_base(n_edges + 1);
  std::vector<int32_t> from_op(n_edges + 1), to_op(n_edges + 1), in_deg(n_ops + 1), out_deg(n_ops + 1),
      order(n_ops + 1);
  std::vector<double> n_sec(sz.num_aux_nodes + 1), n_vol(sz.num_aux_nodes + 1), n_mem(sz.num_aux_nodes + 1);
  aux.edges.resize(sz.num_aux_edges);
  tp_aux_index ix{node_base.data(), edge_base.data(), from_op.data(), to_op.data(),
                  in_deg.data(),    out_deg.data(),   order.data()};
  tp_cost_tensors out{};
  out.node_intra_cost_s = n_sec.data();
  out.node_intra_volume_bytes = n_vol.data();
  out.node_memory_bytes = n_mem.data();
  out.aux_edge_records = aux.edges.data();
  if (minima) {
    minima->row_min_cost_s.assign(sz.num_rows + 1, 0.0);
    minima->row_min_volume_bytes.assign(sz.num_rows + 1, 0.0);
    minima->pair_min_cost_s.assign(n_edges + 1, 0.0);
    minima->pair_min_volume_bytes.assign(n_edges + 1, 0.0);
    out.row_min_cost_s = minima->row_min_cost_s.data();
    out.row_min_volume_bytes = minima->row_min_volume_bytes.data();
    out.edge_pair_min_cost_s = minima->pair_min_cost_s.data();
    out.edge_pair_min_volume_bytes = minima->pair_min_volume_bytes.data();
  }
  clk.mark("output allocation");
  // (the thread's reused device memory: a plan built once needs none of its own)
  detail::check(tp_plan_execute_host_scratch(plan.p, nullptr, &ix, &out));
  clk.mark("execute + D2H");

  if (minima) {
    minima->row_min_cost_s.resize(sz.num_rows);
    minima->row_min_volume_bytes.resize(sz.num_rows);
    minima->pair_min_cost_s.resize(n_edges);
    minima->pair_min_volume_bytes.resize(n_edges);
    minima->edge_from_op.assign(from_op.begin(), from_op.begin() + n_edges);
    minima->edge_to_op.assign(to_op.begin(), to_op.begin() + n_edges);
  }
  aux.topo_order.assign(order.begin(), order.begin() + n_ops);
  aux.in_degree_of.assign(in_deg.begin(), in_deg.begin() + n_ops);
  aux.out_degree_of.assign(out_deg.begin(), out_deg.begin() + n_ops);
  aux.edge_base.resize(n_edges);
  for (int e = 0; e < n_edges; ++e) aux.edge_base[e] = (int)edge_base[e];
  aux.nodes_of_op.resize(n_ops);

  // strategy tables (layout.hpp:270-328), produced by the device enumerator
  std::map<int, std::vector<topoplan::OperatorStrategy>> tables;
  const int64_t N = topo.total_devices();
  for (int i = 0; i < n_ops; ++i) {
    const int p = graph.operators[i].axis_count();
    if (tables.count(p)) continue;
    int64_t S = 0;
    detail::check(tp_enumerate_strategies(p, N, &S, nullptr, nullptr, nullptr, nullptr));
    std::vector<int64_t> deg(S * p), dims(S * p);
    std::vector<int32_t> dmap(S * p), depth(S);
    detail::check(tp_enumerate_strategies(p, N, &S, deg.data(), dmap.data(), dims.data(), depth.data()));
    auto& v = tables[p];
    v.resize(S);
    for (int64_t s = 0; s < S; ++s) {
      v[s].degrees.assign(deg.begin() + s * p, deg.begin() + (s + 1) * p);
      v[s].device_map.assign(dmap.begin() + s * p, dmap.begin() + (s + 1) * p);
      v[s].device_matrix.dims.assign(dims.begin() + s * p, dims.begin() + s * p + depth[s]);
    }
  }
  clk.mark("index + strategy tables");
  aux.nodes.resize(sz.num_aux_nodes);
  // every operator's aux nodes independently (strategy copies and, with
  // layouts, a std::map per node: most of the adapter's host time), on the
  // host's cores for big graphs
  detail::parallel_for(n_ops, sz.num_aux_nodes >= 16384 ? 16 : n_ops + 1, [&](int i) {
    const auto& tab = tables.at(graph.operators[i].axis_count());
    const int64_t S = node_base[i + 1] - node_base[i];
    aux.nodes_of_op[i].resize(S);
    for (int64_t s = 0; s < S; ++s) {
      const int64_t id = node_base[i] + s;
      topoplan::AuxNode& node = aux.nodes[id];
      node.op_index = i;
      node.strategy_index = (int)s;
      node.strategy = tab[s];
      node.strategy.op_id = graph.operators[i].id;
      if (with_layouts) node.layouts = tensor_layouts_b200(graph.operators[i], node.strategy);
      node.intra_cost_s = n_sec[id];
      node.intra_volume_bytes = n_vol[id];
      node.memory_bytes = n_mem[id];
      aux.nodes_of_op[i][s] = (int)id;
    }
  });
  clk.mark(with_layouts ? "nodes + layouts" : "nodes");
  // virtual source edges (aux_graph.hpp:298-312)
  aux.virtual_edge_of_node.assign(aux.nodes.size(), -1);
  for (int i = 0; i < n_ops; ++i) {
    if (aux.in_degree_of[i] != 0) continue;
    for (int node_id : aux.nodes_of_op[i]) {
      const topoplan::AuxNode& node = aux.nodes[node_id];
      topoplan::VirtualEdge ve;
      ve.op_index = i;
      ve.to_node = node_id;
      ve.cost_s = node.intra_cost_s;
      ve.volume_bytes = node.intra_volume_bytes;
      ve.memory_bytes = node.memory_bytes;
      aux.virtual_edge_of_node[node_id] = (int)aux.virtual_edges.size();
      aux.virtual_edges.push_back(ve);
    }
  }
  clk.mark("virtual edges");
  tp_plan_destroy(plan.p);
  plan.p = nullptr;
  clk.mark("plan destroy");
  clk.report();
  return aux;
}

}  // namespace taps_b200

#endif  // TAPS_B200_AUX_GRAPH_B200_HPP_
