// export_b200.hpp — the reference's two on-disk / wire formats of a priced
// auxiliary graph, written directly instead of through intermediate objects.
//
//   std::string lp   = taps_b200::export_lp_b200(aux, mode, device_memory);
//   std::string json = taps_b200::aux_graph_to_json_b200(aux);
//
// export_lp_b200 == topoplan::export_lp(topoplan::formulate(aux, mode,
// device_memory)) (solver.hpp:69-176, 578-600) byte for byte, without the
// IlpProblem (lp_export.hpp does the writing from index arithmetic).
// aux_graph_to_json_b200 == topoplan::aux_graph_to_json(aux).dump()
// (io.hpp:208-239) byte for byte: nlohmann::json's compact dump of the same
// document -- object keys in std::map order, doubles through the library's
// own shortest-round-trip formatter (nlohmann::detail::to_chars, as its
// serializer) -- streamed, without building the Json tree. Needs
// nlohmann/json.hpp (v3.11) on the include path, as io.hpp does.
//
// Both take any topoplan::AuxiliaryGraph: the reference's, or the one
// build_auxiliary_graph_b200 returns (records written by the device).
#ifndef TAPS_B200_EXPORT_B200_HPP_
#define TAPS_B200_EXPORT_B200_HPP_

#include <array>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "topoplan/aux_graph.hpp"
#include "lp_export.hpp"

namespace taps_b200 {

namespace detail {

// The index and SoA view of an AuxiliaryGraph (what the C-ABI returns).
struct AuxArrays {
  std::vector<int64_t> node_base, edge_base;
  std::vector<int32_t> from_op, to_op, in_deg, out_deg;
  std::vector<double> n_sec, n_vol, n_mem, e_sec, e_vol, e_mem;
  LpInput in;

  explicit AuxArrays(const topoplan::AuxiliaryGraph& aux) {
    const int P = (int)aux.nodes_of_op.size(), E = (int)aux.graph.edges.size();
    node_base.assign(P + 1, 0);
    for (int op = 0; op < P; ++op) node_base[op + 1] = node_base[op] + (int64_t)aux.nodes_of_op[op].size();
    edge_base.assign(E + 1, (int64_t)aux.edges.size());
    for (int e = 0; e < E; ++e) edge_base[e] = aux.edge_base[e];
    from_op.resize(E);
    to_op.resize(E);
    for (int e = 0; e < E; ++e) {  // find_op of the endpoints (graph.hpp:135-140)
      from_op[e] = aux.graph.find_op(aux.graph.edges[e].from);
      to_op[e] = aux.graph.find_op(aux.graph.edges[e].to);
    }
    in_deg.assign(aux.in_degree_of.begin(), aux.in_degree_of.end());
    out_deg.assign(aux.out_degree_of.begin(), aux.out_degree_of.end());
    for (const auto& n : aux.nodes) {
      n_sec.push_back(n.intra_cost_s);
      n_vol.push_back(n.intra_volume_bytes);
      n_mem.push_back(n.memory_bytes);
    }
    for (const auto& x : aux.edges) {
      e_sec.push_back(x.cost_s);
      e_vol.push_back(x.volume_bytes);
      e_mem.push_back(x.memory_bytes);
    }
    in = LpInput{P, E, node_base.data(), edge_base.data(), from_op.data(), to_op.data(), in_deg.data(),
                 out_deg.data(), n_sec.data(), n_vol.data(), n_mem.data(), e_sec.data(), e_vol.data(),
                 e_mem.data()};
  }
};

struct StringSink {
  std::string* s;
  void operator()(const char* p, size_t n) { s->append(p, n); }
};

}  // namespace detail

inline std::string export_lp_b200(const topoplan::AuxiliaryGraph& aux, topoplan::CostMode mode,
                                  double device_memory) {
  const detail::AuxArrays a(aux);
  std::string out;
  out.reserve(64 * (aux.edges.size() + aux.nodes.size()) + 4096);
  detail::StringSink sink{&out};
  write_lp(a.in, mode == topoplan::CostMode::kVolume, device_memory, sink);
  return out;
}

#if __has_include(<nlohmann/json.hpp>) || __has_include("json.hpp")
#if __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
#else
#include "json.hpp"
#endif
#define TAPS_B200_HAVE_JSON 1

namespace detail {

class JsonOut {
 public:
  explicit JsonOut(std::string& s) : s_(s) {}
  void raw(const char* p, size_t n) { s_.append(p, n); }
  void raw(const char* p) { s_.append(p); }
  void ch(char c) { s_.push_back(c); }
  void i64(int64_t v) {
    char b[24];
    const auto r = std::to_chars(b, b + sizeof(b), v);
    s_.append(b, (size_t)(r.ptr - b));
  }
  void f64(double v) {  // serializer::dump_float: null for non-finite, else the library's to_chars
    if (!std::isfinite(v)) {
      s_.append("null");
      return;
    }
    char b[64];
    char* end = ::nlohmann::detail::to_chars(b, b + sizeof(b), v);
    s_.append(b, (size_t)(end - b));
  }
  void str(const std::string& v) {  // serializer::dump_escaped, ensure_ascii = false
    s_.push_back('"');
    for (unsigned char c : v) {
      switch (c) {
        case '"': s_.append("\\\""); break;
        case '\\': s_.append("\\\\"); break;
        case '\b': s_.append("\\b"); break;
        case '\f': s_.append("\\f"); break;
        case '\n': s_.append("\\n"); break;
        case '\r': s_.append("\\r"); break;
        case '\t': s_.append("\\t"); break;
        default:
          if (c < 0x20) {
            char b[8];
            std::snprintf(b, sizeof(b), "\\u%04x", (unsigned)c);
            s_.append(b);
          } else {
            s_.push_back((char)c);
          }
      }
    }
    s_.push_back('"');
  }
  template <typename V>
  void ints(const V& v) {
    ch('[');
    for (size_t i = 0; i < v.size(); ++i) {
      if (i) ch(',');
      i64((int64_t)v[i]);
    }
    ch(']');
  }

 private:
  std::string& s_;
};

}  // namespace detail

// topoplan::aux_graph_to_json(aux).dump() (io.hpp:193-239): keys sorted
// (nlohmann::json objects are std::maps), compact separators.
inline std::string aux_graph_to_json_b200(const topoplan::AuxiliaryGraph& aux) {
  std::string s;
  s.reserve(160 * aux.edges.size() + 256 * aux.nodes.size() + 1024);
  detail::JsonOut o(s);
  o.raw("{\"edges\":[");
  for (size_t i = 0; i < aux.edges.size(); ++i) {
    const topoplan::AuxEdge& e = aux.edges[i];
    if (i) o.ch(',');
    o.raw("{\"cost_seconds\":");
    o.f64(e.cost_s);
    o.raw(",\"edge\":");
    o.i64(e.original_edge);
    o.raw(",\"from_node\":");
    o.i64(e.from_node);
    o.raw(",\"memory_bytes\":");
    o.f64(e.memory_bytes);
    o.raw(",\"to_node\":");
    o.i64(e.to_node);
    o.raw(",\"volume_bytes\":");
    o.f64(e.volume_bytes);
    o.ch('}');
  }
  o.raw("],\"nodes\":[");
  for (size_t i = 0; i < aux.nodes.size(); ++i) {
    const topoplan::AuxNode& n = aux.nodes[i];
    const topoplan::OperatorNode& op = aux.graph.operators[n.op_index];
    if (i) o.ch(',');
    o.raw("{\"axes\":[");  // strategy_to_json (io.hpp:193-203) plus the node payload
    for (size_t a = 0; a < op.axes.size(); ++a) {
      if (a) o.ch(',');
      o.str(op.axes[a].name);
    }
    o.raw("],\"degrees\":");
    o.ints(n.strategy.degrees);
    o.raw(",\"device_map\":");
    o.ints(n.strategy.device_map);
    o.raw(",\"device_matrix\":");
    o.ints(n.strategy.device_matrix.dims);
    o.raw(",\"display_matrix\":");
    o.ints(n.strategy.display_matrix());
    o.raw(",\"intra_cost_seconds\":");
    o.f64(n.intra_cost_s);
    o.raw(",\"intra_volume_bytes\":");
    o.f64(n.intra_volume_bytes);
    o.raw(",\"memory_bytes\":");
    o.f64(n.memory_bytes);
    o.raw(",\"op\":");
    o.str(op.id);
    o.ch('}');
  }
  o.raw("],\"schema\":\"topoplan-auxgraph/v1\",\"virtual_edges\":[");
  for (size_t i = 0; i < aux.virtual_edges.size(); ++i) {
    const topoplan::VirtualEdge& e = aux.virtual_edges[i];
    if (i) o.ch(',');
    o.raw("{\"cost_seconds\":");
    o.f64(e.cost_s);
    o.raw(",\"memory_bytes\":");
    o.f64(e.memory_bytes);
    o.raw(",\"op\":");
    o.str(aux.graph.operators[e.op_index].id);
    o.raw(",\"to_node\":");
    o.i64(e.to_node);
    o.raw(",\"volume_bytes\":");
    o.f64(e.volume_bytes);
    o.ch('}');
  }
  o.raw("]}");
  return s;
}
#endif  // json.hpp available

}  // namespace taps_b200

#endif  // TAPS_B200_EXPORT_B200_HPP_
