// lp_export.hpp — the reference's ILP as CPLEX LP text, written straight from
// the cost tensors.
//
// topoplan::export_lp(topoplan::formulate(aux, mode, device_memory))
// (solver.hpp:69-176, 546-600) builds an IlpProblem -- one heap string per
// variable, one term vector per row -- and then prints it. write_lp emits the
// same bytes from the SoA tensors and the build's index alone (what the C-ABI
// returns), without materialising the problem: variable names, row
// membership and coefficients are index arithmetic over node_base /
// edge_base, numbers are "%.17g" (std::to_chars with precision 17 is
// printf's %.17g exactly).
//
// Header-only C++17, no topoplan dependency: used by the engine library
// (tp_plan_export_lp) and by the C++ adapter (export_lp_b200).
#ifndef TAPS_B200_LP_EXPORT_HPP_
#define TAPS_B200_LP_EXPORT_HPP_

#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace taps_b200 {

// One build, as the C-ABI returns it (tp_aux_index + tp_cost_tensors).
struct LpInput {
  int32_t num_ops = 0, num_edges = 0;
  const int64_t* node_base = nullptr;     // [num_ops + 1]
  const int64_t* edge_base = nullptr;     // [num_edges + 1]
  const int32_t* edge_from_op = nullptr;  // [num_edges] find_op(from)
  const int32_t* edge_to_op = nullptr;    // [num_edges] find_op(to)
  const int32_t* in_degree = nullptr;     // [num_ops] by operator id (ComputationGraph::in_degree)
  const int32_t* out_degree = nullptr;    // [num_ops]
  const double *n_sec = nullptr, *n_vol = nullptr, *n_mem = nullptr;  // per aux node
  const double *e_sec = nullptr, *e_vol = nullptr, *e_mem = nullptr;  // per aux edge
};

// Appends text to `out`; `flush(const char*, size_t)` is called whenever the
// buffer passes `chunk` bytes and once at the end (a file, or a string).
template <typename Flush>
class LpWriter {
 public:
  LpWriter(Flush& f, size_t chunk = 1 << 20) : flush_(f), chunk_(chunk) { buf_.reserve(chunk + 256); }
  void put(const char* s, size_t n) {
    buf_.append(s, n);
    if (buf_.size() >= chunk_) drain();
  }
  void put(const char* s) { put(s, std::strlen(s)); }
  void put(char c) {
    buf_.push_back(c);
    if (buf_.size() >= chunk_) drain();
  }
  void num(int64_t v) {
    char b[24];
    const auto r = std::to_chars(b, b + sizeof(b), v);
    put(b, (size_t)(r.ptr - b));
  }
  void coeff(double v) {  // detail::format_coeff (solver.hpp:548-552): "%.17g"
    char b[64];
    if (!std::isfinite(v)) {  // printf's spelling of inf / nan
      put(std::isnan(v) ? (std::signbit(v) ? "-nan" : "nan") : (v < 0 ? "-inf" : "inf"));
      return;
    }
    const auto r = std::to_chars(b, b + sizeof(b), v, std::chars_format::general, 17);
    put(b, (size_t)(r.ptr - b));
  }
  void drain() {
    if (!buf_.empty()) flush_(buf_.data(), buf_.size());
    buf_.clear();
  }

 private:
  Flush& flush_;
  size_t chunk_;
  std::string buf_;
};

namespace lp_detail {

template <typename W>
struct Terms {  // detail::append_terms (solver.hpp:554-571), streamed
  W& w;
  bool first = true;
  template <typename Name>
  void add(double c, Name&& name) {
    if (c == 0) return;
    if (first) {
      if (c < 0) w.put("- ", 2);
      first = false;
    } else {
      w.put(c < 0 ? " - " : " + ", 3);
    }
    const double mag = std::fabs(c);
    if (mag != 1.0) {
      w.coeff(mag);
      w.put(' ');
    }
    name();
  }
};

}  // namespace lp_detail

// export_lp(formulate(aux, volume ? kVolume : kTopology, device_memory)).
template <typename Flush>
void write_lp(const LpInput& in, bool volume, double device_memory, Flush& flush) {
  LpWriter<Flush> w(flush);
  const int32_t P = in.num_ops, E = in.num_edges;
  const int64_t nodes = P ? in.node_base[P] : 0;
  auto S = [&](int op) { return in.node_base[op + 1] - in.node_base[op]; };
  // op of every aux node; graph edges into / out of every operator (find_op
  // endpoints, edge order) -- the reference's in/out edge lists of a node are
  // exactly these edges' aux edges with that strategy, ascending
  std::vector<int32_t> op_of(nodes);
  for (int op = 0; op < P; ++op)
    for (int64_t s = 0; s < S(op); ++s) op_of[in.node_base[op] + s] = op;
  std::vector<int32_t> ib(P + 1, 0), ob(P + 1, 0), il(E), ol(E);
  for (int e = 0; e < E; ++e) ++ib[in.edge_to_op[e] + 1], ++ob[in.edge_from_op[e] + 1];
  for (int op = 0; op < P; ++op) ib[op + 1] += ib[op], ob[op + 1] += ob[op];
  {
    std::vector<int32_t> fi(ib.begin(), ib.end() - 1), fo(ob.begin(), ob.end() - 1);
    for (int e = 0; e < E; ++e) il[fi[in.edge_to_op[e]]++] = e, ol[fo[in.edge_from_op[e]]++] = e;
  }
  auto xname = [&](int op, int64_t s) {
    w.put('x');
    w.num(op);
    w.put('_');
    w.num(s);
  };
  auto bname = [&](int e, int64_t su, int64_t sw) {
    w.put('b');
    w.num(e);
    w.put('_');
    w.num(su);
    w.put('_');
    w.num(sw);
  };
  const double* ew = volume ? in.e_vol : in.e_sec;  // edge_weight_by_mode
  const double* nw = volume ? in.n_vol : in.n_sec;  // virtual_weight_by_mode (a source's node payload)

  w.put(volume ? "\\ topoplan ILP export (mode: volume)\n" : "\\ topoplan ILP export (mode: topology)\n");
  w.put("Minimize\n obj: ");
  {
    lp_detail::Terms<LpWriter<Flush>> t{w};
    for (int op = 0; op < P; ++op)  // X vars: a source's virtual edge weight
      if (in.in_degree[op] == 0)
        for (int64_t s = 0; s < S(op); ++s) t.add(nw[in.node_base[op] + s], [&] { xname(op, s); });
    for (int e = 0; e < E; ++e) {  // B vars, aux edge order
      const int u = in.edge_from_op[e], v = in.edge_to_op[e];
      const int64_t Sw = S(v), b0 = in.edge_base[e];
      for (int64_t su = 0; su < S(u); ++su)
        for (int64_t sw = 0; sw < Sw; ++sw) t.add(ew[b0 + su * Sw + sw], [&] { bname(e, su, sw); });
    }
    if (t.first) {  // "0 " and the first variable (there are no edge variables without node ones)
      w.put("0 ");
      if (nodes > 0) xname(0, 0);
      else w.put('x');
    }
  }
  w.put("\nSubject To\n");
  for (int op = 0; op < P; ++op) {  // onestrat rows
    w.put(" onestrat");
    w.num(op);
    w.put(": ");
    lp_detail::Terms<LpWriter<Flush>> t{w};
    for (int64_t s = 0; s < S(op); ++s) t.add(1.0, [&] { xname(op, s); });
    if (t.first) w.put("0 x", 3);  // cannot occur: every operator has >= 1 strategy
    w.put(" = ");
    w.coeff(1.0);
    w.put('\n');
  }
  for (int64_t node = 0; node < nodes; ++node) {
    const int op = op_of[node];
    const int64_t s = node - in.node_base[op];
    for (int dir = 0; dir < 2; ++dir) {
      const int32_t deg = dir ? in.out_degree[op] : in.in_degree[op];
      if (deg <= 0) continue;
      w.put(dir ? " outdeg" : " indeg");
      w.num(node);
      w.put(": ");
      lp_detail::Terms<LpWriter<Flush>> t{w};
      const int32_t* lst = dir ? ol.data() : il.data();
      const int32_t* bnd = dir ? ob.data() : ib.data();
      for (int k = bnd[op]; k < bnd[op + 1]; ++k) {
        const int e = lst[k];
        const int u = in.edge_from_op[e], v = in.edge_to_op[e];
        if (dir) {
          for (int64_t sw = 0; sw < S(v); ++sw) t.add(1.0, [&] { bname(e, s, sw); });
        } else {
          for (int64_t su = 0; su < S(u); ++su) t.add(1.0, [&] { bname(e, su, s); });
        }
      }
      t.add(-(double)deg, [&] { xname(op, s); });
      w.put(" = ");
      w.coeff(0.0);
      w.put('\n');
    }
  }
  w.put(" mem: ");
  {
    lp_detail::Terms<LpWriter<Flush>> t{w};
    for (int e = 0; e < E; ++e) {
      const int u = in.edge_from_op[e], v = in.edge_to_op[e];
      const int64_t Sw = S(v), b0 = in.edge_base[e];
      for (int64_t su = 0; su < S(u); ++su)
        for (int64_t sw = 0; sw < Sw; ++sw) t.add(in.e_mem[b0 + su * Sw + sw], [&] { bname(e, su, sw); });
    }
    for (int op = 0; op < P; ++op)
      if (in.in_degree[op] == 0)
        for (int64_t s = 0; s < S(op); ++s) t.add(in.n_mem[in.node_base[op] + s], [&] { xname(op, s); });
    if (t.first) {
      w.put("0 ");
      if (nodes > 0) xname(0, 0);
      else w.put('x');
    }
  }
  w.put(" <= ");
  w.coeff(device_memory - 1.0);
  w.put("\nBinaries\n");
  for (int op = 0; op < P; ++op)
    for (int64_t s = 0; s < S(op); ++s) {
      w.put(' ');
      xname(op, s);
      w.put('\n');
    }
  for (int e = 0; e < E; ++e) {
    const int u = in.edge_from_op[e], v = in.edge_to_op[e];
    for (int64_t su = 0; su < S(u); ++su)
      for (int64_t sw = 0; sw < S(v); ++sw) {
        w.put(' ');
        bname(e, su, sw);
        w.put('\n');
      }
  }
  w.put("End\n");
  w.drain();
}

}  // namespace taps_b200

#endif  // TAPS_B200_LP_EXPORT_HPP_
