// export_parity.cpp — TEST INFRASTRUCTURE ONLY.
//
// Pins the direct writers of include/taps_b200/export_b200.hpp to the
// reference on the CPU: for graphs built by the UNMODIFIED reference
// (build_auxiliary_graph, included from /root/reference at build time),
//   export_lp_b200(aux, mode, mem)  == export_lp(formulate(aux, mode, mem))   (solver.hpp:578-600)
//   aux_graph_to_json_b200(aux)     == aux_graph_to_json(aux).dump()           (io.hpp:208-239)
// byte for byte, both cost modes; prints the time of each. Built by
// oracle/Makefile into oracle/_ref/export_parity (needs nlohmann/json.hpp,
// the reference's own io.hpp dependency); run by tests/test_export.py.
#include <chrono>
#include <cstdio>
#include <random>
#include <string>

#include "topoplan/aux_graph.hpp"
#include "topoplan/io.hpp"
#include "topoplan/models.hpp"
#include "topoplan/solver.hpp"
#include "test_support.hpp"
#include "taps_b200/export_b200.hpp"

using namespace topoplan;

namespace {
int failures = 0;

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

std::string first_diff(const std::string& a, const std::string& b) {
  size_t i = 0;
  while (i < a.size() && i < b.size() && a[i] == b[i]) ++i;
  return "at byte " + std::to_string(i) + ": '" + a.substr(i > 20 ? i - 20 : 0, 60) + "' vs '" +
         b.substr(i > 20 ? i - 20 : 0, 60) + "'";
}

void check(const std::string& name, const ComputationGraph& g, const ClusterTopology& t, bool json = true) {
  const AuxiliaryGraph aux = build_auxiliary_graph(g, t);
  std::string err;
  double t_ref = 0, t_b200 = 0;
  for (CostMode mode : {CostMode::kTopology, CostMode::kVolume}) {
    auto t0 = std::chrono::steady_clock::now();
    const std::string a = export_lp(formulate(aux, mode, t.device_memory));
    t_ref += ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    const std::string b = taps_b200::export_lp_b200(aux, mode, t.device_memory);
    t_b200 += ms_since(t0);
    if (a != b && err.empty()) err = std::string("export_lp differs (") + to_string(mode) + ") " + first_diff(a, b);
  }
  double j_ref = 0, j_b200 = 0;
  if (json && err.empty()) {
    auto t0 = std::chrono::steady_clock::now();
    const std::string a = aux_graph_to_json(aux).dump();
    j_ref = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    const std::string b = taps_b200::aux_graph_to_json_b200(aux);
    j_b200 = ms_since(t0);
    if (a != b) err = "aux_graph_to_json differs " + first_diff(a, b);
  }
  std::printf("[EXPORT] %-32s %s %zu aux edges; export_lp x2 %.1f ms vs b200 %.1f ms; json %.1f ms vs b200 %.1f ms%s%s\n",
              name.c_str(), err.empty() ? "PASS" : "FAIL", aux.edges.size(), t_ref, t_b200, j_ref, j_b200,
              err.empty() ? "" : ": ", err.c_str());
  std::fflush(stdout);
  if (!err.empty()) ++failures;
}
}  // namespace

int main(int argc, char** argv) {
  const bool big = argc > 1 && std::string(argv[1]) == "--big";
  {
    ComputationGraph g;
    g.operators.push_back(testing::matmul_op("fc1", 256, 1024, 4096, "x0", "x1"));
    g.operators.push_back(testing::elementwise_op("relu", {"x1"}, "x2", 256, 4096));
    g.operators.push_back(testing::matmul_op("fc2", 256, 4096, 1024, "x2", "x3"));
    g.edges = {{"fc1", "relu", "x1"}, {"relu", "fc2", "x2"}};
    check("cfg1 sample graph 2x4", g, {2, 4, 60e9, 6e9, 32e9});
  }
  {
    ComputationGraph one;
    one.operators.push_back(testing::matmul_op("fc", 8, 8, 8));
    check("single op single device", one, {1, 1, 60e9, 60e9, 32e9});
    ComputationGraph chain;
    chain.operators.push_back(testing::matmul_op("fc1", 16, 16, 16, "x0", "x1"));
    chain.operators.push_back(testing::matmul_op("fc2", 16, 16, 16, "x1", "x2"));
    chain.edges.push_back({"fc1", "fc2", "x1"});
    check("two-matmul chain 2x2", chain, {2, 2, 60e9, 6e9, 32e9});
    ComputationGraph empty;
    check("empty graph", empty, {1, 4, 60e9, 60e9, 32e9});
  }
  for (const char* spec : {"alexnet-like", "mlp-chain", "transformer-layer"})
    check(spec, build_graph(parse_model_spec(spec)), {2, 8, 60e9, 6e9, 256e9});
  {
    ModelConfig c2;
    c2.family = ModelFamily::kTransformerLayer;
    c2.hidden = 4096;
    c2.batch = 8;
    c2.seq = 512;
    check("cfg2 transformer h4096 4x8", build_graph(c2), {4, 8, 60e9, 6e9, 80e9});
  }
  {
    std::mt19937 rng(77);
    for (int i = 0; i < 30; ++i) {
      const auto inst = testing::random_planning_instance(rng, 6, 2e5);
      try {
        check("random planning instance " + std::to_string(i), inst.graph, inst.topo);
      } catch (const std::exception&) {  // the reference throws on this instance: nothing to export
      }
    }
  }
  if (big) {  // cfg3-size graphs: LP only on 8x8 (the reference's JSON dump of 335k edges is slow)
    ModelConfig c;
    c.family = ModelFamily::kMlpChain;
    c.layers = 16;
    c.hidden = 4096;
    c.batch = 256;
    check("mlp-chain L16 h4096 8x8", build_graph(c), {8, 8, 60e9, 6e9, 80e9});
  }
  std::printf("[EXPORT] %s (%d failures)\n", failures ? "FAILED" : "ALL PASS", failures);
  return failures ? 1 : 0;
}
