// models_b200.hpp — the input step of the BASELINE workloads for C++ callers:
// graph composers on top of the reference's one-layer builders.
//
//   topoplan::ComputationGraph g = taps_b200::gpt_chain(96, 12288, 8, 2048);     // cfg4
//   std::vector<taps_b200::Scenario> sweep = taps_b200::scenario_sweep(1000);   // cfg5
//
// The reference builds ONE transformer layer (models.hpp:125-197); its paper
// workloads chain layers. gpt_chain composes L copies of that layer: operator
// ids and tensor names of layer l are prefixed "L<l>.", layer l's input x is
// layer l-1's residual output (add2_out), and an edge add2 -> ln1 joins
// consecutive layers. scenario_sweep draws the cfg5 sweep from
// std::mt19937_64(0x230104285) in the draw order of SURVEY.md §8d (family,
// node count, bandwidth ratio, then the family's parameters), so its
// 1,000 scenarios are the ones the Python composer (models.py) and the bench
// use: 16,957,929 aux edges in total. Validation stays the reference's own
// (graph.hpp validate_graph / validate_or_throw).
#ifndef TAPS_B200_MODELS_B200_HPP_
#define TAPS_B200_MODELS_B200_HPP_

#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <vector>

#include "topoplan/graph.hpp"
#include "topoplan/models.hpp"

namespace taps_b200 {

// L chained pre-norm transformer layers (hidden, batch, seq as ModelConfig).
inline topoplan::ComputationGraph gpt_chain(int layers, int64_t hidden, int64_t batch, int64_t seq) {
  topoplan::ModelConfig cfg;
  cfg.family = topoplan::ModelFamily::kTransformerLayer;
  cfg.hidden = hidden;
  cfg.batch = batch;
  cfg.seq = seq;
  const topoplan::ComputationGraph layer = topoplan::build_transformer_layer(cfg);
  topoplan::ComputationGraph g;
  g.operators.reserve(layer.operators.size() * layers);
  g.edges.reserve((layer.edges.size() + 1) * layers);
  std::string x = "x";  // the layer's input tensor
  for (int l = 0; l < layers; ++l) {
    const std::string p = "L" + std::to_string(l) + ".";
    auto ren = [&](const std::string& n) { return n == "x" ? x : p + n; };
    for (topoplan::OperatorNode op : layer.operators) {
      op.id = p + op.id;
      for (auto& t : op.inputs) t.name = ren(t.name);
      for (auto& t : op.outputs) t.name = ren(t.name);
      for (auto& a : op.axes)
        for (auto& s : a.slices) s.tensor = ren(s.tensor);
      g.operators.push_back(std::move(op));
    }
    if (l > 0) g.edges.push_back({"L" + std::to_string(l - 1) + ".add2", p + "ln1", x});
    for (const topoplan::GraphEdge& e : layer.edges) g.edges.push_back({p + e.from, p + e.to, ren(e.tensor)});
    x = p + "add2_out";
  }
  return g;
}

struct Scenario {
  std::string family;  // "mlp-chain", "transformer-layer", "alexnet-like", "gpt-chain"
  topoplan::ComputationGraph graph;
  topoplan::ClusterTopology topo;
  double ratio = 1;  // intra / inter bandwidth
};

// cfg5: `count` (model, mesh, bandwidth-ratio) scenarios.
inline std::vector<Scenario> scenario_sweep(int count = 1000, uint64_t seed = 0x230104285ull) {
  std::mt19937_64 rng(seed);
  std::vector<Scenario> out;
  out.reserve(count);
  for (int i = 0; i < count; ++i) {
    Scenario s;
    const uint64_t fam = rng() % 4;
    const int nodes = 1 << (rng() % 4);
    s.ratio = std::pow(10.0, static_cast<double>(rng() % 1001) / 500.0);
    topoplan::ModelConfig c;
    if (fam == 0) {
      c.family = topoplan::ModelFamily::kMlpChain;
      c.layers = 2 + static_cast<int64_t>(rng() % 7);
      c.hidden = static_cast<int64_t>(256) << (rng() % 5);
      c.batch = 256;
      s.graph = topoplan::build_graph(c);
      s.family = "mlp-chain";
    } else if (fam == 1) {
      c.family = topoplan::ModelFamily::kTransformerLayer;
      c.hidden = static_cast<int64_t>(1024) << (rng() % 3);
      c.batch = 8;
      c.seq = 512;
      s.graph = topoplan::build_graph(c);
      s.family = "transformer-layer";
    } else if (fam == 2) {
      c.family = topoplan::ModelFamily::kAlexnetLike;
      c.batch = 64;
      s.graph = topoplan::build_graph(c);
      s.family = "alexnet-like";
    } else {
      const int L = 2 + static_cast<int>(rng() % 3);
      s.graph = gpt_chain(L, 2048, 8, 512);
      s.family = "gpt-chain";
    }
    s.topo = topoplan::ClusterTopology{nodes, 8, 60e9, 60e9 / s.ratio, 80e9};
    out.push_back(std::move(s));
  }
  return out;
}

// The other BASELINE configurations.
inline topoplan::ClusterTopology cfg3_topology(int nodes, double ratio = 10) {
  return topoplan::ClusterTopology{nodes, 8, 60e9, 60e9 / ratio, 80e9};
}
inline topoplan::ComputationGraph cfg3_graph() { return gpt_chain(24, 2048, 8, 512); }
inline topoplan::ComputationGraph cfg4_graph() { return gpt_chain(96, 12288, 8, 2048); }
inline topoplan::ClusterTopology cfg4_topology(double ratio = 10) {
  return topoplan::ClusterTopology{16, 8, 60e9, 60e9 / ratio, 80e9};
}

}  // namespace taps_b200

#endif  // TAPS_B200_MODELS_B200_HPP_
