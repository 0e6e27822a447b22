// The four unit solvers of the reference's library API
// (proj/include/levelrank/solvers.hpp:31-54: solve_singletons, solve_cac,
// solve_small_scc, solve_large_scc), run on the GPU through the same level
// loop as compute_pagerank.  A unit is solved as a graph of its own: its
// vertices (local ids 0..m-1, same order), its edges, and for every vertex
// enough extra out-edges to fresh sink vertices that its walk out-degree (and
// self-loop flag) equals the one in the full graph -- so every push factor
// c/deg is the reference's.  Sinks never push back, so the unit's values are
// those of the unit solve; small_threshold forces the SCC kind (m + 1 for
// SccSmall, 1 for SccLarge), and the power series reports its iterations.
#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "levelrank/engine.hpp"
#include "lr_cuda.h"

namespace levelrank {
inline namespace b200 {
namespace {

std::vector<double> solve_as_graph(const Graph& g, const SolveUnit& unit, std::span<const double> w_local,
                                   const SolverParams& params, VertexId threshold, std::int64_t* iterations,
                                   int device) {
  validate_params(params);
  const VertexId m = unit.size();
  if (static_cast<VertexId>(w_local.size()) != m)
    throw std::invalid_argument("weight vector does not match the unit size");
  if (iterations) *iterations = 0;
  if (m == 0) return {};
  std::vector<VertexId> intra(static_cast<std::size_t>(m), 0);
  std::vector<VertexId> src, dst;
  src.reserve(unit.edges.size());
  dst.reserve(unit.edges.size());
  for (const auto& [a, b] : unit.edges) {
    if (a < 0 || a >= m || b < 0 || b >= m) throw std::invalid_argument("unit edge out of range");
    if (a == b) continue;  // self-loops follow the graph's flag below
    src.push_back(a);
    dst.push_back(b);
    ++intra[static_cast<std::size_t>(a)];
  }
  VertexId next = m;
  for (VertexId a = 0; a < m; ++a) {
    const VertexId v = unit.global_ids[static_cast<std::size_t>(a)];
    if (v < 0 || v >= g.vertex_count()) throw std::invalid_argument("unit vertex out of range");
    if (g.has_loop(v)) {
      src.push_back(a);
      dst.push_back(a);
    }
    const VertexId extra = g.out_degree(v) - (g.has_loop(v) ? 1 : 0) - intra[static_cast<std::size_t>(a)];
    if (extra < 0) throw std::invalid_argument("unit edges exceed the vertex's out-degree");
    for (VertexId k = 0; k < extra; ++k) {
      src.push_back(a);
      dst.push_back(next++);
    }
  }
  const Graph sub = Graph::from_edge_arrays(next, src.data(), dst.data(), static_cast<EdgeId>(src.size()),
                                            g.loop_policy());
  std::vector<double> w(static_cast<std::size_t>(next), 0.0);
  std::copy(w_local.begin(), w_local.end(), w.begin());
  EngineResult res = compute_pagerank(sub, w, params, ExecutionMode::Sequential, threshold, 0, device);
  if (iterations)
    for (const UnitRecord& u : res.report.units) *iterations = std::max(*iterations, u.iterations);
  res.ranks.resize(static_cast<std::size_t>(m));
  return res.ranks;
}

}  // namespace

std::vector<double> solve_singletons(const Graph& g, const SolveUnit& unit, std::span<const double> w_local,
                                     const SolverParams& params, int device) {
  if (!unit.edges.empty() &&
      std::any_of(unit.edges.begin(), unit.edges.end(), [](const auto& e) { return e.first != e.second; }))
    throw std::invalid_argument("a singleton group has no edges between its vertices");
  return solve_as_graph(g, unit, w_local, params, 100, nullptr, device);
}

std::vector<double> solve_cac(const Graph& g, const SolveUnit& unit, std::span<const double> w_local,
                              const SolverParams& params, EdgeId* edge_visits, int device) {
  // solvers.cpp:84-85: a unit that is not acyclic never drains its queue
  const VertexId m = unit.size();
  std::vector<VertexId> indeg(static_cast<std::size_t>(m), 0), off(static_cast<std::size_t>(m) + 1, 0), adj;
  EdgeId visits = 0;
  for (const auto& [a, b] : unit.edges)
    if (a != b && a >= 0 && a < m && b >= 0 && b < m) ++off[static_cast<std::size_t>(a) + 1], ++indeg[static_cast<std::size_t>(b)], ++visits;
  for (VertexId i = 0; i < m; ++i) off[static_cast<std::size_t>(i) + 1] += off[static_cast<std::size_t>(i)];
  adj.resize(static_cast<std::size_t>(off[static_cast<std::size_t>(m)]));
  {
    std::vector<VertexId> cur(off.begin(), off.end() - 1);
    for (const auto& [a, b] : unit.edges)
      if (a != b && a >= 0 && a < m && b >= 0 && b < m) adj[static_cast<std::size_t>(cur[static_cast<std::size_t>(a)]++)] = b;
  }
  std::vector<VertexId> queue;
  for (VertexId i = 0; i < m; ++i)
    if (indeg[static_cast<std::size_t>(i)] == 0) queue.push_back(i);
  for (std::size_t h = 0; h < queue.size(); ++h)
    for (VertexId k = off[static_cast<std::size_t>(queue[h])]; k < off[static_cast<std::size_t>(queue[h]) + 1]; ++k)
      if (--indeg[static_cast<std::size_t>(adj[static_cast<std::size_t>(k)])] == 0) queue.push_back(adj[static_cast<std::size_t>(k)]);
  if (static_cast<VertexId>(queue.size()) != m) throw CycleError("cycle inside an acyclic component");
  if (g.loop_policy() == LoopPolicy::Keep)
    for (const VertexId v : unit.global_ids) visits += g.has_loop(v) ? 1 : 0;
  std::vector<double> r = solve_as_graph(g, unit, w_local, params, 100, nullptr, device);
  if (edge_visits) *edge_visits = visits;
  return r;
}

std::vector<double> solve_small_scc(const Graph& g, const SolveUnit& unit, std::span<const double> w_local,
                                    const SolverParams& params, int device) {
  return solve_as_graph(g, unit, w_local, params, unit.size() + 1, nullptr, device);
}

std::vector<double> solve_large_scc(const Graph& g, const SolveUnit& unit, std::span<const double> w_local,
                                    const SolverParams& params, std::int64_t& iterations, PowerSeriesStats* stats,
                                    int device) {
  if (!stats) return solve_as_graph(g, unit, w_local, params, 1, &iterations, device);
  validate_params(params);
  const VertexId m = unit.size();
  if (static_cast<VertexId>(w_local.size()) != m)
    throw std::invalid_argument("weight vector does not match the unit size");
  // pull CSR: row b's sources a in ascending order = solve_large_scc's
  // accumulation order over unit.edges (sorted by source, then target)
  const bool keep = g.loop_policy() == LoopPolicy::Keep;
  std::vector<std::pair<VertexId, VertexId>> e;
  e.reserve(unit.edges.size());
  for (const auto& [a, b] : unit.edges) {
    if (a < 0 || a >= m || b < 0 || b >= m) throw std::invalid_argument("unit edge out of range");
    if (a == b && !keep) continue;
    e.emplace_back(b, a);
  }
  std::stable_sort(e.begin(), e.end());
  std::vector<long long> ptr(static_cast<std::size_t>(m) + 1, 0);
  std::vector<std::int32_t> src(e.size());
  for (std::size_t k = 0; k < e.size(); ++k) {
    ++ptr[static_cast<std::size_t>(e[k].first) + 1];
    src[k] = e[k].second;
  }
  for (VertexId i = 0; i < m; ++i) ptr[static_cast<std::size_t>(i) + 1] += ptr[static_cast<std::size_t>(i)];
  std::vector<double> pf(static_cast<std::size_t>(m));
  for (VertexId i = 0; i < m; ++i)
    pf[static_cast<std::size_t>(i)] = params.c / static_cast<double>(g.walk_out_degree(unit.global_ids[static_cast<std::size_t>(i)]));
  const std::int64_t cap = iteration_cap(params);
  std::vector<double> ranks(static_cast<std::size_t>(m)), l1(static_cast<std::size_t>(cap) + 1);
  double mn = 0.0;
  const lr_status st = lr_series_stats_csr(device, m, ptr.data(), src.data(), pf.data(), w_local.data(), params.tol,
                                           cap, ranks.data(), &iterations, l1.data(),
                                           static_cast<std::int64_t>(l1.size()), &mn);
  if (st != LR_OK) {
    const std::string msg = lr_last_error();
    if (st == LR_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
  l1.resize(static_cast<std::size_t>(std::min<std::int64_t>(iterations, static_cast<std::int64_t>(l1.size()))));
  stats->increment_l1_norms = std::move(l1);
  stats->min_increment_entry = m > 0 ? mn : 0.0;
  return ranks;
}

}  // namespace b200
}  // namespace levelrank

