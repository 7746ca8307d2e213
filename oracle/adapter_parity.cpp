// adapter_parity.cpp — TEST INFRASTRUCTURE ONLY.
//
// Runs the reference's build_auxiliary_graph (the UNMODIFIED headers from
// /root/reference, included at build time) and the B200 drop-in
// taps_b200::build_auxiliary_graph_b200 on the same inputs and checks that
// every field of the two topoplan::AuxiliaryGraph objects is identical
// (costs bit-for-bit), then that the reference's own ILP solver
// (formulate + solve, solver.hpp:69-493) selects the same strategies with
// the same objective on both, that price_assignment agrees and that
// export_lp emits the same text. Built by oracle/Makefile into
// oracle/_ref/adapter_parity; run on a GPU box by tests/test_gpu_adapter.py.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "topoplan/aux_graph.hpp"
#include "topoplan/models.hpp"
#include "topoplan/solver.hpp"
#include "test_support.hpp"  // the reference's test oracles, -I$(REF_TESTS) (see Makefile)
#include "topoplan/io.hpp"  // aux_graph_to_json (needs nlohmann/json.hpp, -I in oracle/Makefile)
#include "taps_b200/aux_graph_b200.hpp"
#include "taps_b200/export_b200.hpp"
#include "taps_b200/models_b200.hpp"
#include "taps_b200/solver_b200.hpp"

using namespace topoplan;

namespace {

int failures = 0;

bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof(double)) == 0; }

std::string compare(const AuxiliaryGraph& r, const AuxiliaryGraph& g) {
  if (r.nodes.size() != g.nodes.size()) return "node count";
  if (r.edges.size() != g.edges.size()) return "edge count";
  if (r.virtual_edges.size() != g.virtual_edges.size()) return "virtual edge count";
  if (r.topo_order != g.topo_order) return "topo_order";
  if (r.edge_base != g.edge_base) return "edge_base";
  if (r.in_degree_of != g.in_degree_of || r.out_degree_of != g.out_degree_of) return "degrees";
  if (r.nodes_of_op != g.nodes_of_op) return "nodes_of_op";
  if (r.virtual_edge_of_node != g.virtual_edge_of_node) return "virtual_edge_of_node";
  for (std::size_t i = 0; i < r.nodes.size(); ++i) {
    const AuxNode &a = r.nodes[i], &b = g.nodes[i];
    if (a.op_index != b.op_index || a.strategy_index != b.strategy_index) return "node index " + std::to_string(i);
    if (!(a.strategy == b.strategy) || !(a.strategy.device_matrix == b.strategy.device_matrix) ||
        a.strategy.op_id != b.strategy.op_id)
      return "node strategy " + std::to_string(i);
    if (!same_bits(a.intra_cost_s, b.intra_cost_s) || !same_bits(a.intra_volume_bytes, b.intra_volume_bytes) ||
        !same_bits(a.memory_bytes, b.memory_bytes))
      return "node payload " + std::to_string(i);
    // AuxNode::layouts: the adapter's own tensor_layouts_b200 against derive_tensor_layouts
    if (a.layouts.size() != b.layouts.size()) return "node layouts " + std::to_string(i);
    for (auto ia = a.layouts.begin(), ib = b.layouts.begin(); ia != a.layouts.end(); ++ia, ++ib) {
      const TensorLayout &x = ia->second, &y = ib->second;
      if (ia->first != ib->first || x.spec.name != y.spec.name || x.spec.shape != y.spec.shape ||
          x.spec.element_size != y.spec.element_size || x.matrix.dims != y.matrix.dims ||
          x.map.entries != y.map.entries)
        return "node layouts " + std::to_string(i);
    }
  }
  for (std::size_t e = 0; e < r.edges.size(); ++e) {
    const AuxEdge &a = r.edges[e], &b = g.edges[e];
    if (a.original_edge != b.original_edge || a.from_node != b.from_node || a.to_node != b.to_node)
      return "edge index " + std::to_string(e);
    if (!same_bits(a.cost_s, b.cost_s) || !same_bits(a.volume_bytes, b.volume_bytes) ||
        !same_bits(a.memory_bytes, b.memory_bytes))
      return "edge payload " + std::to_string(e);
  }
  for (std::size_t v = 0; v < r.virtual_edges.size(); ++v) {
    const VirtualEdge &a = r.virtual_edges[v], &b = g.virtual_edges[v];
    if (a.op_index != b.op_index || a.to_node != b.to_node || !same_bits(a.cost_s, b.cost_s) ||
        !same_bits(a.volume_bytes, b.volume_bytes) || !same_bits(a.memory_bytes, b.memory_bytes))
      return "virtual edge " + std::to_string(v);
  }
  return "";
}

void report(const std::string& name, const std::string& err, const std::string& extra = "") {
  std::printf("[PARITY] %-34s %s%s%s\n", name.c_str(), err.empty() ? "PASS  " : "FAIL: ", "",
              err.empty() ? extra.c_str() : err.c_str());
  std::fflush(stdout);
  if (!err.empty()) ++failures;
}

struct SolveCfg {
  bool solve = false;
  int threads = 8;
  std::int64_t max_nodes = 200'000'000;
};

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

void check_case(const std::string& name, const ComputationGraph& graph, const ClusterTopology& topo,
                SolveCfg sc = {}) {
  AuxiliaryGraph ref, gpu;
  taps_b200::SolverMinima minima;
  std::string ref_err, gpu_err;
  double t_build_ref = 0, t_build_b200 = 0;
  try {
    const auto t0 = std::chrono::steady_clock::now();
    ref = build_auxiliary_graph(graph, topo);
    t_build_ref = ms_since(t0);
  } catch (const Error& e) {
    ref_err = "Error";
  } catch (const std::out_of_range& e) {
    ref_err = "out_of_range";
  }
  try {
    const auto t0 = std::chrono::steady_clock::now();
    gpu = taps_b200::build_auxiliary_graph_b200(graph, topo, CostMode::kTopology, -1, true, &minima);
    t_build_b200 = ms_since(t0);
  } catch (const Error& e) {
    gpu_err = "Error";
  } catch (const std::out_of_range& e) {
    gpu_err = "out_of_range";
  }
  if (!ref_err.empty() || !gpu_err.empty()) {
    report(name, ref_err == gpu_err ? "" : "reference threw '" + ref_err + "', b200 threw '" + gpu_err + "'",
           "both throw " + ref_err);
    return;
  }
  std::string err = compare(ref, gpu);
  // edge_weight (aux_graph.hpp:184) through the adapter's layouts
  if (err.empty() && !ref.edges.empty()) {
    const EdgeWeight a = edge_weight(ref.graph, 0, ref.nodes[ref.edges[0].from_node],
                                     ref.nodes[ref.edges[0].to_node], topo);
    const EdgeWeight b = edge_weight(gpu.graph, 0, gpu.nodes[gpu.edges[0].from_node],
                                     gpu.nodes[gpu.edges[0].to_node], topo);
    if (!same_bits(a.cost_s, b.cost_s)) err = "edge_weight via layouts";
  }
  // the solver's search context (solver.hpp:218-287) from the device minima
  for (CostMode mode : {CostMode::kTopology, CostMode::kVolume}) {
    if (!err.empty()) break;
    const detail::SearchContext a = detail::make_context(ref, mode, topo.device_memory);
    const detail::SearchContext b = taps_b200::make_context_b200(gpu, minima, mode, topo.device_memory);
    auto same_vec = [](const std::vector<double>& x, const std::vector<double>& y) {
      if (x.size() != y.size()) return false;
      for (std::size_t i = 0; i < x.size(); ++i)
        if (!same_bits(x[i], y[i])) return false;
      return true;
    };
    bool ok = a.order == b.order && a.pos_of_op == b.pos_of_op && a.in_edges_of == b.in_edges_of &&
              a.cond_min.size() == b.cond_min.size() && same_vec(a.pair_min, b.pair_min) &&
              same_vec(a.source_min, b.source_min) && same_vec(a.suffix_mem_min, b.suffix_mem_min) &&
              same_vec(a.virtual_min_mem, b.virtual_min_mem) && same_bits(a.root_bound, b.root_bound) &&
              same_bits(a.memory_bound, b.memory_bound) && a.mode == b.mode;
    for (std::size_t e = 0; ok && e < a.cond_min.size(); ++e) ok = same_vec(a.cond_min[e], b.cond_min[e]);
    if (!ok) err = std::string("make_context_b200 differs (") + to_string(mode) + ")";
  }
  // formulate_b200 against the reference's formulate (solver.hpp:69-176), field by field
  double t_ref_ms = 0, t_b200_ms = 0;
  for (CostMode mode : {CostMode::kTopology, CostMode::kVolume}) {
    if (!err.empty()) break;
    const auto t0 = std::chrono::steady_clock::now();
    const IlpProblem a = formulate(ref, mode, topo.device_memory);
    const auto t1 = std::chrono::steady_clock::now();
    const IlpProblem b = taps_b200::formulate_b200(gpu, mode, topo.device_memory);
    const auto t2 = std::chrono::steady_clock::now();
    t_ref_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
    t_b200_ms += std::chrono::duration<double, std::milli>(t2 - t1).count();
    bool ok = a.mode == b.mode && same_bits(a.memory_bound, b.memory_bound) && a.vars.size() == b.vars.size() &&
              a.objective.size() == b.objective.size() && a.rows.size() == b.rows.size() &&
              a.x_var_of_node == b.x_var_of_node && a.b_var_of_edge == b.b_var_of_edge;
    for (std::size_t i = 0; ok && i < a.vars.size(); ++i) {
      const auto &x = a.vars[i], &y = b.vars[i];
      ok = x.kind == y.kind && x.name == y.name && x.op_index == y.op_index &&
           x.strategy_index == y.strategy_index && x.edge_id == y.edge_id && same_bits(a.objective[i], b.objective[i]);
    }
    for (std::size_t i = 0; ok && i < a.rows.size(); ++i) {
      const auto &x = a.rows[i], &y = b.rows[i];
      ok = x.name == y.name && x.is_equality == y.is_equality && same_bits(x.rhs, y.rhs) &&
           x.terms.size() == y.terms.size();
      for (std::size_t k = 0; ok && k < x.terms.size(); ++k)
        ok = x.terms[k].first == y.terms[k].first && same_bits(x.terms[k].second, y.terms[k].second);
    }
    if (!ok) err = std::string("formulate_b200 differs (") + to_string(mode) + ")";
  }
  // the wire formats of the GPU-built graph (export_b200.hpp) against the
  // reference's on its own graph: export_lp of both modes; the JSON dump
  // (below ~0.4M aux edges: nlohmann's tree of a cfg4 graph takes many GB)
  double t_lp_ref = 0, t_lp_b200 = 0, t_js_ref = 0, t_js_b200 = 0;
  for (CostMode mode : {CostMode::kTopology, CostMode::kVolume}) {
    if (!err.empty()) break;
    auto t0 = std::chrono::steady_clock::now();
    const std::string a = export_lp(formulate(ref, mode, topo.device_memory));
    t_lp_ref += ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    const std::string b = taps_b200::export_lp_b200(gpu, mode, topo.device_memory);
    t_lp_b200 += ms_since(t0);
    if (a != b) err = std::string("export_lp_b200 differs (") + to_string(mode) + ")";
  }
  if (err.empty() && gpu.edges.size() <= 400000) {
    auto t0 = std::chrono::steady_clock::now();
    const std::string a = aux_graph_to_json(ref).dump();
    t_js_ref = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    const std::string b = taps_b200::aux_graph_to_json_b200(gpu);
    t_js_b200 = ms_since(t0);
    if (a != b) err = "aux_graph_to_json_b200 differs";
  } else if (err.empty()) {
    const auto t0 = std::chrono::steady_clock::now();
    const std::string b = taps_b200::aux_graph_to_json_b200(gpu);
    t_js_b200 = ms_since(t0);
    std::printf("[PARITY]   %s: aux_graph_to_json_b200 %.1f ms, %.1f MB (reference dump not built at this size)\n",
                name.c_str(), t_js_b200, b.size() / 1e6);
  }
  std::string extra = std::to_string(gpu.edges.size()) + " aux edges bit-identical";
  if (gpu.edges.size() >= 100000) {
    char buf[400];
    std::snprintf(buf, sizeof(buf),
                  "; build_auxiliary_graph %.1f ms vs build_auxiliary_graph_b200 %.1f ms; formulate x2 modes %.1f ms, "
                  "formulate_b200 %.1f ms; export_lp x2 %.1f ms vs export_lp_b200 %.1f ms; json %.1f vs %.1f ms",
                  t_build_ref, t_build_b200, t_ref_ms, t_b200_ms, t_lp_ref, t_lp_b200, t_js_ref, t_js_b200);
    extra += buf;
  }
  if (err.empty() && sc.solve) {
    for (CostMode mode : {CostMode::kTopology, CostMode::kVolume}) {
      SolveOptions opts;
      opts.threads = sc.threads;
      opts.max_nodes = sc.max_nodes;
      const PlanSolution a = solve(formulate(ref, mode, topo.device_memory), opts);
      const PlanSolution b = solve(formulate(gpu, mode, topo.device_memory), opts);
      if (a.feasible != b.feasible || a.strategy_per_op != b.strategy_per_op || !same_bits(a.objective, b.objective) ||
          a.optimal != b.optimal) {
        err = std::string("ILP differs (") + to_string(mode) + ")";
        break;
      }
      if (export_lp(formulate(ref, mode, topo.device_memory)) != export_lp(formulate(gpu, mode, topo.device_memory))) {
        err = std::string("export_lp differs (") + to_string(mode) + ")";
        break;
      }
      char buf[200];
      std::snprintf(buf, sizeof(buf), "; ILP %s obj %.17g %s (%lld nodes)", to_string(mode), a.objective,
                    a.optimal ? "optimal" : "budget", (long long)a.nodes_explored);
      extra += buf;
    }
    std::mt19937 rng(7);
    for (int t = 0; err.empty() && t < 50; ++t) {
      std::vector<int> asg(graph.operators.size());
      for (std::size_t i = 0; i < asg.size(); ++i) asg[i] = (int)(rng() % ref.strategies_of((int)i));
      for (CostMode mode : {CostMode::kTopology, CostMode::kVolume}) {
        const AssignmentPrice a = price_assignment(ref, asg, mode), b = price_assignment(gpu, asg, mode);
        if (!same_bits(a.cost, b.cost) || !same_bits(a.memory_bytes, b.memory_bytes)) err = "price_assignment";
      }
    }
  }
  report(name, err, extra);
}

// cfg5: the seeded scenario sweep (SURVEY.md §8d draw order). For every
// sampled scenario both builds go through the reference's own ILP in both
// cost modes and run_compare's TAPS-vs-volume ratio (pipeline.hpp:152-168:
// both winners priced in topology mode) must be bit-identical.
void check_sweep(int count, int every) {
  // the C++ composer (include/taps_b200/models_b200.hpp); every scenario built
  // on the GPU (the aux-edge total of SURVEY §8d), every `every`-th also by the reference
  const std::vector<taps_b200::Scenario> sweep = taps_b200::scenario_sweep(count);
  int checked = 0;
  std::int64_t total = 0;
  for (int i = 0; i < count; ++i) {
    const ComputationGraph& g = sweep[i].graph;
    const ClusterTopology& topo = sweep[i].topo;
    const int nodes = topo.node_count;
    const double ratio = sweep[i].ratio;
    std::string name = sweep[i].family;
    if (i % every != 0) {
      total += (std::int64_t)taps_b200::build_auxiliary_graph_b200(g, topo).edges.size();
      continue;
    }
    const AuxiliaryGraph ref = build_auxiliary_graph(g, topo);
    const AuxiliaryGraph gpu = taps_b200::build_auxiliary_graph_b200(g, topo, CostMode::kTopology, -1, true);
    total += (std::int64_t)gpu.edges.size();
    std::string err = compare(ref, gpu);
    double ratios[2] = {0, 0};
    const AuxiliaryGraph* both[2] = {&ref, &gpu};
    for (int k = 0; err.empty() && k < 2; ++k) {
      SolveOptions opts;
      opts.threads = 1;
      opts.max_nodes = 20000;  // fixed budget, one thread: a deterministic search
      const PlanSolution v = solve(formulate(*both[k], CostMode::kVolume, topo.device_memory), opts);
      const PlanSolution t = solve(formulate(*both[k], CostMode::kTopology, topo.device_memory), opts);
      const double den = price_assignment(*both[k], v.strategy_per_op, CostMode::kTopology).cost;
      const double num = price_assignment(*both[k], t.strategy_per_op, CostMode::kTopology).cost;
      ratios[k] = den == 0 ? 1.0 : num / den;
      static PlanSolution keep_v, keep_t;
      if (k == 0) {
        keep_v = v;
        keep_t = t;
      } else if (keep_v.strategy_per_op != v.strategy_per_op || keep_t.strategy_per_op != t.strategy_per_op ||
                 !same_bits(keep_v.objective, v.objective) || !same_bits(keep_t.objective, t.objective)) {
        err = "ILP selection differs";
      }
    }
    if (err.empty() && !same_bits(ratios[0], ratios[1])) err = "TAPS/volume ratio differs";
    char buf[200];
    std::snprintf(buf, sizeof(buf), "%zu aux edges, %dx8, ratio bw %.3g: TAPS/volume %.4f", gpu.edges.size(), nodes,
                  ratio, ratios[0]);
    report("cfg5 #" + std::to_string(i) + " " + name, err, buf);
    ++checked;
  }
  std::printf("[PARITY] cfg5 sweep: %d scenarios checked, %lld aux edges over all %d\n", checked, (long long)total,
              count);
  if (count == 1000 && total != 16957929) {
    std::printf("[PARITY] cfg5 sweep aux-edge total differs from SURVEY 8d's 16957929\n");
    ++failures;
  }
}

}  // namespace

// --time: the C++ drop-in on cfg4 (with and without AuxNode::layouts), best of 3, and the
// reference's build once; no parity checks (TAPS_B200_PROFILE=1 adds the adapter's phases).
int time_cfg4() {
  const ComputationGraph g = taps_b200::gpt_chain(96, 12288, 8, 2048);
  const ClusterTopology topo{16, 8, 60e9, 6e9, 80e9};
  for (int layouts = 0; layouts < 2; ++layouts) {
    double best = 1e30;
    for (int r = 0; r < 3; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      const AuxiliaryGraph a = taps_b200::build_auxiliary_graph_b200(g, topo, CostMode::kTopology, -1, layouts != 0);
      best = std::min(best, ms_since(t0));
      if (a.edges.size() != 2155580u) return 1;
    }
    std::printf("[TIME] cfg4 build_auxiliary_graph_b200 (layouts %d): %.1f ms (best of 3)\n", layouts, best);
  }
  const auto t0 = std::chrono::steady_clock::now();
  const AuxiliaryGraph ref = build_auxiliary_graph(g, topo);
  std::printf("[TIME] cfg4 build_auxiliary_graph (reference, one thread): %.1f ms\n", ms_since(t0));
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "--time") return time_cfg4();
  const bool big = argc > 1 && std::string(argv[1]) == "--big";  // every 10th cfg5 scenario instead of every 40th
  const ClusterTopology t2x4{2, 4, 60e9, 6e9, 32e9};
  {  // cfg1: data/sample_graph.json on 2 x 4
    ComputationGraph g;
    g.operators.push_back(testing::matmul_op("fc1", 256, 1024, 4096, "x0", "x1"));
    g.operators.push_back(testing::elementwise_op("relu", {"x1"}, "x2", 256, 4096));
    g.operators.push_back(testing::matmul_op("fc2", 256, 4096, 1024, "x2", "x3"));
    g.edges = {{"fc1", "relu", "x1"}, {"relu", "fc2", "x2"}};
    check_case("cfg1 sample graph 2x4", g, t2x4, SolveCfg{true});
  }
  {
    ComputationGraph chain;
    chain.operators.push_back(testing::matmul_op("fc1", 16, 16, 16, "x0", "x1"));
    chain.operators.push_back(testing::matmul_op("fc2", 16, 16, 16, "x1", "x2"));
    chain.edges.push_back({"fc1", "fc2", "x1"});
    check_case("two-matmul chain 1x4", chain, {1, 4, 60e9, 60e9, 32e9}, SolveCfg{true});
    check_case("two-matmul chain 2x2", chain, {2, 2, 60e9, 6e9, 32e9}, SolveCfg{true});
    ComputationGraph one;
    one.operators.push_back(testing::matmul_op("fc", 8, 8, 8));
    check_case("single op single device", one, {1, 1, 60e9, 60e9, 32e9}, SolveCfg{true});
    ComputationGraph bad;
    bad.operators.push_back(testing::matmul_op("fc", 6, 6, 6));
    check_case("indivisible shapes throw", bad, {1, 4, 60e9, 60e9, 32e9});
    ComputationGraph dangling = chain;
    dangling.edges.push_back({"fc2", "nope", "x2"});
    check_case("dangling edge throws", dangling, {1, 4, 60e9, 60e9, 32e9});
    ComputationGraph missing = chain;
    missing.edges.push_back({"fc1", "fc2", "nope"});
    check_case("missing edge tensor throws", missing, {1, 4, 60e9, 60e9, 32e9});
  }
  {
    ModelConfig tl;
    tl.family = ModelFamily::kTransformerLayer;
    tl.hidden = 256;
    tl.seq = 64;
    tl.batch = 4;
    check_case("transformer-layer h256 2x4", build_graph(tl), {2, 4, 60e9, 6e9, 80e9}, SolveCfg{true});
    check_case("alexnet-like 2x8", build_graph(parse_model_spec("alexnet-like")), {2, 8, 60e9, 6e9, 256e9},
               SolveCfg{true});
    check_case("mlp-chain 4x8", build_graph(parse_model_spec("mlp-chain")), {4, 8, 60e9, 6e9, 256e9},
               SolveCfg{true});
    ModelConfig c2;
    c2.family = ModelFamily::kTransformerLayer;
    c2.hidden = 4096;
    c2.batch = 8;
    c2.seq = 512;
    check_case("cfg2 transformer h4096 4x8", build_graph(c2), {4, 8, 60e9, 6e9, 80e9}, SolveCfg{true, 16});
  }
  {
    std::mt19937 rng(4096);
    for (int i = 0; i < 40; ++i) {
      const auto inst = testing::random_planning_instance(rng, 6, 2e5);
      check_case("random planning instance " + std::to_string(i), inst.graph, inst.topo, SolveCfg{i % 4 == 0});
    }
  }
  {  // cfg3 (24 layers) on 2/4/8 x 8 and cfg4 (96 layers, 16 x 8) with a fixed node
     // budget and threads=1: a deterministic truncated search, so the
     // selections, objectives, `optimal` flags and LP texts must be identical
    const ComputationGraph gpt24 = taps_b200::gpt_chain(24, 2048, 8, 512);
    check_case("cfg3 GPT-24 h2048 2x8", gpt24, {2, 8, 60e9, 6e9, 80e9}, SolveCfg{true, 1, 200000});
    check_case("cfg3 GPT-24 h2048 4x8", gpt24, {4, 8, 60e9, 6e9, 80e9}, SolveCfg{true, 1, 20000});
    check_case("cfg3 GPT-24 h2048 8x8 r100", gpt24, {8, 8, 60e9, 0.6e9, 80e9}, SolveCfg{true, 1, 20000});
    check_case("cfg4 GPT-96 h12288 16x8", taps_b200::gpt_chain(96, 12288, 8, 2048), {16, 8, 60e9, 6e9, 80e9},
               SolveCfg{true, 1, 5000});
  }
  check_sweep(1000, big ? 10 : 40);
  std::printf("[PARITY] %s (%d failures)\n", failures ? "FAILED" : "ALL PASS", failures);
  return failures ? 1 : 0;
}
