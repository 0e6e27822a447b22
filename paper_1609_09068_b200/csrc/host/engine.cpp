// C++ engine API (include/levelrank/engine.hpp) over the C-ABI.  The solve is
// always the GPU level loop; any failure surfaces as the reference's
// exception types (engine.cpp:92-97, solvers.cpp:11-15,84-85,103-106,159).
#include "levelrank/engine.hpp"

#include <algorithm>
#include <chrono>
#include <stdexcept>
#include <string>

#include "lr_cuda.h"
#include "plan_internal.hpp"

namespace levelrank {
inline namespace b200 {
namespace detail {
lr_status baseline_solve(const Graph& g, const double* w, int64_t wn, double c, double tol, int device, double* ranks,
                         double* r1, lr_report* rep);
}
namespace {

[[noreturn]] void raise(lr_status st) {
  const std::string msg = lr_last_error();
  switch (st) {
    case LR_EINVAL:
      throw std::invalid_argument(msg);
    case LR_ECYCLE:
      throw std::logic_error(msg);
    case LR_EIO:
      throw IoError(msg);
    default:
      throw std::runtime_error(msg);
  }
}
void check(lr_status st) {
  if (st != LR_OK) raise(st);
}

}  // namespace

void validate_params(const SolverParams& params) { check(lr_validate_params(params.c, params.tol)); }

std::int64_t iteration_cap(const SolverParams& params) { return lr_iteration_cap(params.c, params.tol); }

ErrorBound error_bound(std::int64_t large, std::int64_t n, const SolverParams& params) {
  double o[2];
  lr_error_bound(large, n, params.c, params.tol, o);
  return {o[0], o[1]};
}

void propagate_weights(std::span<const CrossEdge> cross, std::span<const double> ranks, double c,
                       std::span<double> weights, int device) {
  std::vector<std::int32_t> s(cross.size()), d(cross.size()), g(cross.size());
  for (std::size_t i = 0; i < cross.size(); ++i) {
    s[i] = cross[i].src;
    d[i] = cross[i].dst;
    g[i] = cross[i].src_out_degree;
  }
  // ranks are indexed by source, weights by destination: the two vectors may
  // differ in length (engine.cpp:83-87); the C-ABI takes one length
  const std::size_t nmax = std::max(ranks.size(), weights.size());
  if (ranks.size() == weights.size()) {
    check(lr_propagate_weights(device, s.data(), d.data(), g.data(), static_cast<std::int64_t>(cross.size()),
                               ranks.data(), static_cast<std::int64_t>(ranks.size()), c, weights.data()));
    return;
  }
  std::vector<double> r(nmax, 0.0), w(nmax, 0.0);
  std::copy(ranks.begin(), ranks.end(), r.begin());
  std::copy(weights.begin(), weights.end(), w.begin());
  for (std::size_t i = 0; i < cross.size(); ++i)
    if (static_cast<std::size_t>(d[i]) >= weights.size() || static_cast<std::size_t>(s[i]) >= ranks.size())
      throw std::invalid_argument("cross edge out of range");
  check(lr_propagate_weights(device, s.data(), d.data(), g.data(), static_cast<std::int64_t>(cross.size()), r.data(),
                             static_cast<std::int64_t>(nmax), c, w.data()));
  std::copy(w.begin(), w.begin() + static_cast<std::ptrdiff_t>(weights.size()), weights.begin());
}

struct PageRankEngine::Impl {
  const Graph* g = nullptr;
  Partition p;
  Layout L;
  lr_ctx* ctx = nullptr;
  VertexId threshold = 100;
  int device = 0;
  lr_census census{};
  double plan_ms = 0.0, upload_ms = 0.0;
  ~Impl() {
    if (ctx) lr_ctx_free(ctx);
  }
};

PageRankEngine::PageRankEngine(const Graph& g, VertexId small_threshold, int device) : impl_(new Impl) {
  if (small_threshold < 1) throw std::invalid_argument("small_threshold must be at least 1");
  impl_->g = &g;
  impl_->threshold = small_threshold;
  impl_->device = device;
  const auto t0 = std::chrono::steady_clock::now();
  {
    detail::InEdges in;
    impl_->p = detail::find_components_with_in_edges(g, nullptr, in);
    impl_->L = detail::build_layout_from(g, impl_->p, small_threshold, in);
  }
  const PartitionCensus c = census(impl_->p);
  impl_->census = lr_census{c.components, c.scc_components, c.cac_components, c.singleton_cacs, c.largest_component,
                            c.largest_kind == ComponentKind::Scc, c.max_level, c.level_count};
  const auto t1 = std::chrono::steady_clock::now();
  impl_->plan_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  check(lr_ctx_create(device, &impl_->ctx));
  const Layout& L = impl_->L;
  lr_layout lay{L.n,
                L.level_count(),
                L.keep_loops,
                L.unit_count(),
                static_cast<std::int64_t>(L.xsrc.size()),
                static_cast<std::int64_t>(L.isrc.size()),
                static_cast<std::int64_t>(L.depth_ptr.size()),
                L.level_row_begin.data(),
                L.level_unit_begin.data(),
                L.vertex_of.data(),
                L.row_of.data(),
                L.deg.data(),
                L.loop.data(),
                L.xptr.data(),
                L.xsrc.data(),
                L.iptr.data(),
                L.isrc.data(),
                L.unit_kind.data(),
                L.unit_level.data(),
                L.unit_row_begin.data(),
                L.unit_edges.data(),
                L.cac_depth_begin.data(),
                L.depth_ptr.data()};
  check(lr_ctx_upload(impl_->ctx, &lay));
  impl_->upload_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
}

PageRankEngine::~PageRankEngine() = default;

const Layout& PageRankEngine::layout() const { return impl_->L; }
const Partition& PageRankEngine::partition() const { return impl_->p; }

EngineResult PageRankEngine::solve(std::span<const double> weights, const SolverParams& params, ExecutionMode mode,
                                   int threads) {
  validate_params(params);
  const Graph& g = *impl_->g;
  const VertexId n = g.vertex_count();
  if (static_cast<std::int64_t>(weights.size()) != n)
    throw std::invalid_argument("weight vector does not match the vertex count");
  for (const double x : weights)
    if (x < 0.0) throw std::invalid_argument("weights must be non-negative");
  const auto t0 = std::chrono::steady_clock::now();
  EngineResult res;
  SolveReport& rep = res.report;
  rep.mode = mode == ExecutionMode::Parallel ? "parallel" : "sequential";
  rep.threads = mode == ExecutionMode::Parallel ? (threads > 0 ? threads : host_threads()) : 1;
  rep.c = params.c;
  rep.tol = params.tol;
  rep.keep_loops = g.loop_policy() == LoopPolicy::Keep;
  rep.small_threshold = impl_->threshold;
  rep.vertices = n;
  rep.edges = g.edge_count();
  rep.device = impl_->device;
  res.ranks.assign(static_cast<std::size_t>(n), 0.0);
  if (n == 0) return res;
  double wmax = 0.0;
  for (const double x : weights) wmax = std::max(wmax, x);
  rep.all_weights_zero = wmax == 0.0;
  const lr_census& c = impl_->census;
  rep.components = c.components;
  rep.scc_components = c.scc_components;
  rep.cac_components = c.cac_components;
  rep.singleton_cacs = c.singleton_cacs;
  rep.largest_component = c.largest_component;
  rep.largest_component_kind = c.largest_is_scc ? "scc" : "cac";
  rep.max_level = c.max_level;
  rep.level_count = c.level_count;
  rep.plan_ms = impl_->plan_ms;
  rep.upload_ms = impl_->upload_ms;

  const Layout& L = impl_->L;
  std::vector<std::int64_t> iters(static_cast<std::size_t>(L.unit_count()), 0);
  res.r1.assign(static_cast<std::size_t>(n), 0.0);
  lr_solve_info info{};
  check(lr_solve(impl_->ctx, weights.data(), params.c, params.tol, res.ranks.data(), res.r1.data(), &info,
                 iters.data()));
  if (rep.all_weights_zero) res.r1.clear();
  rep.device_ms = info.device_ms;
  rep.cross_edge_count = L.cross_edge_count;
  rep.units.resize(static_cast<std::size_t>(L.unit_count()));
  std::vector<double> unit_ms(rep.units.size(), 0.0);  // LR_UNIT_TIMES=1: device span per unit
  if (!unit_ms.empty() && lr_ctx_unit_times(impl_->ctx, unit_ms.data(), static_cast<std::int64_t>(unit_ms.size())) != LR_OK)
    std::fill(unit_ms.begin(), unit_ms.end(), 0.0);
  for (std::size_t u = 0; u < rep.units.size(); ++u) {
    UnitRecord& r = rep.units[u];
    r.kind = static_cast<UnitKind>(L.unit_kind[u]);
    r.level = L.unit_level[u];
    r.size = L.unit_row_begin[u + 1] - L.unit_row_begin[u];
    r.edges = L.unit_edges[u];
    r.iterations = iters[u];
    r.wall_ms = unit_ms[u];
    rep.total_iterations += r.iterations;
    if (r.kind == UnitKind::SccLarge) {
      rep.iterative_edge_work += r.iterations * r.edges;
      rep.iterative_edges += r.edges;
      rep.large_scc_vertices += r.size;
    } else {
      rep.single_pass_edge_work += r.edges;
    }
  }
  rep.single_pass_edge_work += L.cross_edge_count;
  rep.total_edge_work = rep.iterative_edge_work + rep.single_pass_edge_work;
  rep.mean_iterations_per_edge = rep.iterative_edges > 0 ? static_cast<double>(rep.iterative_edge_work) /
                                                               static_cast<double>(rep.iterative_edges)
                                                         : 0.0;
  const ErrorBound b = error_bound(rep.large_scc_vertices, n, params);
  rep.eps_tot = b.eps_tot;
  rep.eps_avg = b.eps_avg;
  rep.solve_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  rep.wall_ms = rep.plan_ms + rep.upload_ms + rep.solve_ms;
  return res;
}

EngineResult compute_pagerank(const Graph& g, std::span<const double> weights, const SolverParams& params,
                              ExecutionMode mode, VertexId small_threshold, int threads, int device) {
  validate_params(params);
  if (static_cast<std::int64_t>(weights.size()) != g.vertex_count())
    throw std::invalid_argument("weight vector does not match the vertex count");
  for (const double x : weights)
    if (x < 0.0) throw std::invalid_argument("weights must be non-negative");
  if (g.vertex_count() == 0) {
    EngineResult res;
    res.report.vertices = 0;
    res.report.mode = mode == ExecutionMode::Parallel ? "parallel" : "sequential";
    return res;
  }
  PageRankEngine eng(g, small_threshold, device);
  return eng.solve(weights, params, mode, threads);
}

EngineResult compute_baseline(const Graph& g, std::span<const double> weights, const SolverParams& params,
                              int device) {
  validate_params(params);
  const VertexId n = g.vertex_count();
  if (static_cast<std::int64_t>(weights.size()) != n)
    throw std::invalid_argument("weight vector does not match the vertex count");
  EngineResult res;
  res.ranks.assign(static_cast<std::size_t>(n), 0.0);
  res.r1.assign(static_cast<std::size_t>(n), 0.0);
  lr_report r{};
  check(detail::baseline_solve(g, weights.data(), static_cast<std::int64_t>(weights.size()), params.c, params.tol,
                               device, res.ranks.data(), res.r1.data(), &r));
  SolveReport& rep = res.report;  // engine.cpp:194-216
  rep.method = "baseline";
  rep.c = params.c;
  rep.tol = params.tol;
  rep.keep_loops = g.loop_policy() == LoopPolicy::Keep;
  rep.vertices = n;
  rep.edges = g.edge_count();
  rep.all_weights_zero = r.all_weights_zero != 0;
  rep.total_iterations = r.total_iterations;
  rep.iterative_edge_work = r.iterative_edge_work;
  rep.iterative_edges = r.iterative_edges;
  rep.total_edge_work = r.total_edge_work;
  rep.mean_iterations_per_edge = r.mean_iterations_per_edge;
  rep.wall_ms = r.wall_ms;
  rep.plan_ms = r.plan_ms;
  rep.upload_ms = r.upload_ms;
  rep.solve_ms = r.solve_ms;
  rep.device_ms = r.device_ms;
  rep.device = device;
  if (rep.all_weights_zero || n == 0) res.r1.clear();
  return res;
}

}  // namespace b200
}  // namespace levelrank
