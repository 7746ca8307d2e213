// solver_b200.hpp — the solver's search context from device-computed minima.
//
//   taps_b200::SolverMinima m;
//   topoplan::AuxiliaryGraph aux = taps_b200::build_auxiliary_graph_b200(g, topo, mode, -1, false, &m);
//   topoplan::detail::SearchContext ctx = taps_b200::make_context_b200(aux, m, mode, memory_bound);
//
// make_context_b200 returns exactly what topoplan::detail::make_context
// (solver.hpp:218-287) returns — every field bit-identical (checked by
// oracle/adapter_parity.cpp) — but takes cond_min and pair_min, its
// O(|E_A|) part, from the device (rowmin_kernel / pairmin_kernel) instead of
// rescanning every aux edge on the host, and the edge endpoints from the
// build's index instead of find_op's linear scans. What is left on the host is
// O(|V_A| + |E|): positions, in-edge lists, source minima, the suffix memory
// floor and the root bound, summed in the reference's order (edges ascending,
// then sources in operator order).
#ifndef TAPS_B200_SOLVER_B200_HPP_
#define TAPS_B200_SOLVER_B200_HPP_

#include <algorithm>
#include <limits>
#include <vector>

#include "topoplan/solver.hpp"
#include "aux_graph_b200.hpp"

namespace taps_b200 {

inline topoplan::detail::SearchContext make_context_b200(const topoplan::AuxiliaryGraph& aux,
                                                         const SolverMinima& m, topoplan::CostMode mode,
                                                         double memory_bound) {
  topoplan::detail::SearchContext ctx;
  ctx.aux = &aux;
  ctx.mode = mode;
  ctx.memory_bound = memory_bound;
  ctx.order = aux.topo_order;
  const int n_ops = (int)aux.graph.operators.size();
  const int n_edges = (int)aux.graph.edges.size();
  ctx.pos_of_op.assign(n_ops, -1);
  for (int t = 0; t < (int)ctx.order.size(); ++t) ctx.pos_of_op[ctx.order[t]] = t;

  // cond_min / pair_min: device rows, edge-major, S(producer) rows per edge
  const bool volume = mode == topoplan::CostMode::kVolume;
  const std::vector<double>& rows = volume ? m.row_min_volume_bytes : m.row_min_cost_s;
  const std::vector<double>& pairs = volume ? m.pair_min_volume_bytes : m.pair_min_cost_s;
  ctx.in_edges_of.resize(n_ops);
  ctx.cond_min.resize(n_edges);
  ctx.pair_min.assign(pairs.begin(), pairs.begin() + n_edges);
  std::size_t r = 0;
  for (int e = 0; e < n_edges; ++e) {
    ctx.in_edges_of[m.edge_to_op[e]].push_back(e);
    const std::size_t su_n = (std::size_t)aux.strategies_of(m.edge_from_op[e]);
    ctx.cond_min[e].assign(rows.begin() + r, rows.begin() + r + su_n);
    r += su_n;
  }

  const double inf = std::numeric_limits<double>::infinity();
  ctx.source_min.assign(n_ops, 0.0);
  ctx.virtual_min_mem.assign(n_ops, 0.0);
  for (int op = 0; op < n_ops; ++op) {
    double src = inf, mem = inf;
    for (int id : aux.nodes_of_op[op]) {
      mem = std::min(mem, aux.nodes[id].memory_bytes);
      if (aux.in_degree_of[op] == 0)
        src = std::min(src, aux.virtual_weight_by_mode(aux.virtual_edges[aux.virtual_edge_of_node[id]], mode));
    }
    if (aux.in_degree_of[op] == 0) ctx.source_min[op] = src;
    ctx.virtual_min_mem[op] = mem;
  }
  ctx.suffix_mem_min.assign(ctx.order.size() + 1, 0.0);
  for (int t = (int)ctx.order.size() - 1; t >= 0; --t)
    ctx.suffix_mem_min[t] = ctx.suffix_mem_min[t + 1] + ctx.virtual_min_mem[ctx.order[t]];

  double root = 0;
  for (int e = 0; e < n_edges; ++e) root += ctx.pair_min[e];
  for (int op = 0; op < n_ops; ++op)
    if (aux.in_degree_of[op] == 0) root += ctx.source_min[op];
  ctx.root_bound = root;
  return ctx;
}

}  // namespace taps_b200

#endif  // TAPS_B200_SOLVER_B200_HPP_
