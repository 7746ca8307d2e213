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
#include <string>
#include <unordered_map>
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

// topoplan::formulate (solver.hpp:69-176) on a graph built by
// build_auxiliary_graph_b200: the same IlpProblem (variables, names,
// objective bits, rows and terms in the same order; export_lp byte-identical,
// checked by oracle/adapter_parity.cpp), assembled from the cost tensors' index
// arithmetic instead of per-node edge lists: aux node ids are contiguous per
// operator (node = node_base[op] + s) and aux edge ids are (edge, su, sw)
// row-major, so the in-edges of node (w, sw) are edge_base[e] + su*|Sw| + sw for
// the in-edges e of w ascending and su ascending — already the ascending aux-id
// order the reference's push_back loop produces.
inline topoplan::IlpProblem formulate_b200(const topoplan::AuxiliaryGraph& aux, topoplan::CostMode mode,
                                           double device_memory) {
  using topoplan::IlpProblem;
  IlpProblem problem;
  problem.aux = &aux;
  problem.mode = mode;
  problem.memory_bound = device_memory;
  const int n_ops = (int)aux.nodes_of_op.size();
  const int n_edges = (int)aux.graph.edges.size();
  const std::size_t n_nodes = aux.nodes.size(), n_aux = aux.edges.size();

  // find_op (graph.hpp:135-140): the first operator with the id
  std::unordered_map<std::string, int> first_op;
  for (int i = 0; i < (int)aux.graph.operators.size(); ++i) first_op.emplace(aux.graph.operators[i].id, i);
  std::vector<int> from_op(n_edges), to_op(n_edges);
  std::vector<std::vector<int>> in_of(n_ops), out_of(n_ops);
  for (int e = 0; e < n_edges; ++e) {
    from_op[e] = first_op.at(aux.graph.edges[e].from);
    to_op[e] = first_op.at(aux.graph.edges[e].to);
    in_of[to_op[e]].push_back(e);
    out_of[from_op[e]].push_back(e);
  }

  problem.vars.resize(n_nodes + n_aux);
  problem.x_var_of_node.assign(n_nodes, -1);
  int v = 0;
  for (int op = 0; op < n_ops; ++op) {
    for (int node_id : aux.nodes_of_op[op]) {
      IlpProblem::Var& var = problem.vars[v];
      var.kind = IlpProblem::Var::Kind::kNode;
      var.op_index = op;
      var.strategy_index = aux.nodes[node_id].strategy_index;
      var.name = "x" + std::to_string(op) + "_" + std::to_string(var.strategy_index);
      problem.x_var_of_node[node_id] = v++;
    }
  }
  problem.b_var_of_edge.resize(n_aux);
  problem.objective.assign(n_nodes + n_aux, 0.0);
  for (int e = 0; e < n_edges; ++e) {
    const int Su = aux.strategies_of(from_op[e]), Sw = aux.strategies_of(to_op[e]);
    const std::string prefix = "b" + std::to_string(e) + "_";
    std::size_t id = (std::size_t)aux.edge_base[e];
    for (int su = 0; su < Su; ++su) {
      const std::string pre_su = prefix + std::to_string(su) + "_";
      for (int sw = 0; sw < Sw; ++sw, ++id) {
        IlpProblem::Var& var = problem.vars[v];
        var.kind = IlpProblem::Var::Kind::kEdge;
        var.edge_id = (int)id;
        var.name = pre_su + std::to_string(sw);
        problem.b_var_of_edge[id] = v;
        problem.objective[v++] = aux.edge_weight_by_mode(aux.edges[id], mode);
      }
    }
  }
  for (const topoplan::VirtualEdge& ve : aux.virtual_edges)
    problem.objective[problem.x_var_of_node[ve.to_node]] = aux.virtual_weight_by_mode(ve, mode);

  problem.rows.reserve(n_ops + 2 * n_nodes + 1);
  for (int op = 0; op < n_ops; ++op) {
    IlpProblem::Row row;
    row.name = "onestrat" + std::to_string(op);
    row.terms.reserve(aux.nodes_of_op[op].size());
    for (int node_id : aux.nodes_of_op[op]) row.terms.push_back({problem.x_var_of_node[node_id], 1.0});
    row.is_equality = true;
    row.rhs = 1.0;
    problem.rows.push_back(std::move(row));
  }
  for (std::size_t node_id = 0; node_id < n_nodes; ++node_id) {
    const int op = aux.nodes[node_id].op_index;
    const int s = aux.nodes[node_id].strategy_index;
    const int x = problem.x_var_of_node[node_id];
    if (aux.in_degree_of[op] > 0) {  // aux edges into (op, s)
      IlpProblem::Row row;
      row.name = "indeg" + std::to_string(node_id);
      for (int e : in_of[op]) {
        const int Su = aux.strategies_of(from_op[e]), Sw = aux.strategies_of(op);
        for (int su = 0; su < Su; ++su)
          row.terms.push_back({problem.b_var_of_edge[(std::size_t)aux.edge_base[e] + (std::size_t)su * Sw + s], 1.0});
      }
      row.terms.push_back({x, -static_cast<double>(aux.in_degree_of[op])});
      row.is_equality = true;
      row.rhs = 0.0;
      problem.rows.push_back(std::move(row));
    }
    if (aux.out_degree_of[op] > 0) {  // aux edges out of (op, s)
      IlpProblem::Row row;
      row.name = "outdeg" + std::to_string(node_id);
      for (int e : out_of[op]) {
        const int Sw = aux.strategies_of(to_op[e]);
        const std::size_t base = (std::size_t)aux.edge_base[e] + (std::size_t)s * Sw;
        for (int sw = 0; sw < Sw; ++sw) row.terms.push_back({problem.b_var_of_edge[base + sw], 1.0});
      }
      row.terms.push_back({x, -static_cast<double>(aux.out_degree_of[op])});
      row.is_equality = true;
      row.rhs = 0.0;
      problem.rows.push_back(std::move(row));
    }
  }
  IlpProblem::Row mem;
  mem.name = "mem";
  for (std::size_t e = 0; e < n_aux; ++e)
    if (aux.edges[e].memory_bytes != 0) mem.terms.push_back({problem.b_var_of_edge[e], aux.edges[e].memory_bytes});
  for (const topoplan::VirtualEdge& ve : aux.virtual_edges)
    if (ve.memory_bytes != 0) mem.terms.push_back({problem.x_var_of_node[ve.to_node], ve.memory_bytes});
  mem.is_equality = false;
  mem.rhs = device_memory - 1.0;
  problem.rows.push_back(std::move(mem));
  return problem;
}

}  // namespace taps_b200

#endif  // TAPS_B200_SOLVER_B200_HPP_
