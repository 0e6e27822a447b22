// extern "C" host half of include/lr_cuda.h: graph, partition, plan
// (partition + layout), generators, solver helpers, and the one-call
// lr_compute_pagerank.  Every C++ exception is caught here and mapped to a
// status code; nothing throws across the ABI.
#include <chrono>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <cmath>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>

#include "levelrank/engine.hpp"
#include "levelrank/graph.hpp"
#include "levelrank/partition.hpp"
#include "levelrank/schedule.hpp"
#include "lr_cuda.h"
#include "plan_internal.hpp"

namespace levelrank {
inline namespace b200 {
namespace gen {
Graph rmat(std::int32_t scale, std::int64_t edge_factor, double a, double b, double c, std::uint64_t seed);
Graph dangle(const Graph& g, double p, std::uint64_t seed);
Graph planted(VertexId n, std::int32_t n_scc, std::int32_t smin, std::int32_t smax, std::int64_t budget,
              double out_degree, std::int64_t inter_edges, double dangling_fraction, std::uint64_t seed);
Graph deep_dag(std::int32_t levels, std::int32_t width, std::int32_t smin, std::int32_t smax, double scc_out_degree,
               std::int32_t bmin, std::int32_t bmax, double inter_out_degree, std::int32_t reach, std::uint64_t seed);
}  // namespace gen
}  // namespace b200
}  // namespace levelrank

namespace lrerr {
thread_local std::string g_msg;
void set(const std::string& msg) { g_msg = msg; }
}  // namespace lrerr

struct lr_graph {
  levelrank::Graph g;
};

struct lr_plan {
  const levelrank::Graph* g = nullptr;
  levelrank::Partition p;
  levelrank::Layout L;
  std::int32_t threshold = 100;
  bool baseline = false;                       // whole graph as one unit (no partition, no schedule)
  std::unique_ptr<levelrank::Schedule> sched;  // built lazily for parity views
  std::vector<std::int32_t> flat_ids_cache;
};

namespace {

using namespace levelrank;

lr_status from_exception() {
  try {
    throw;
  } catch (const ParseError& e) {
    lrerr::set(e.what());
    return LR_EIO;
  } catch (const IoError& e) {
    lrerr::set(e.what());
    return LR_EIO;
  } catch (const std::invalid_argument& e) {
    lrerr::set(e.what());
    return LR_EINVAL;
  } catch (const CycleError& e) {
    lrerr::set(e.what());
    return LR_ECYCLE;
  } catch (const std::length_error& e) {
    lrerr::set(std::string("out of host memory: ") + e.what());
    return LR_ENOMEM;
  } catch (const std::logic_error& e) {  // out_of_range, domain_error, internal consistency checks
    lrerr::set(e.what());
    return LR_EINVAL;
  } catch (const std::bad_alloc&) {
    lrerr::set("out of host memory");
    return LR_ENOMEM;
  } catch (const std::exception& e) {
    lrerr::set(e.what());
    return LR_ECUDA;
  }
}

template <typename F>
lr_status guarded(F&& f) {
  try {
    f();
    return LR_OK;
  } catch (...) {
    return from_exception();
  }
}

lr_status wrap_graph(Graph&& g, lr_graph** out) {
  *out = new lr_graph{std::move(g)};
  return LR_OK;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* lr_last_error(void) { return lrerr::g_msg.c_str(); }
const char* lr_version(void) { return "levelrank-b200 0.1 (sm_100a)"; }

lr_status lr_graph_from_edges(int32_t n, const int32_t* src, const int32_t* dst, int64_t m, int keep_loops,
                              lr_graph** out) {
  *out = nullptr;
  return guarded([&] {
    wrap_graph(Graph::from_edge_arrays(n, src, dst, m, keep_loops ? LoopPolicy::Keep : LoopPolicy::Ignore), out);
  });
}

lr_status lr_graph_from_csr(int32_t n, const int64_t* offsets, const int32_t* targets, int keep_loops,
                            lr_graph** out) {
  *out = nullptr;
  return guarded([&] {
    if (n < 0) throw std::invalid_argument("vertex count must be non-negative");
    std::vector<EdgeId> off(offsets, offsets + n + 1);
    std::vector<VertexId> tgt(targets, targets + (n >= 0 ? offsets[n] : 0));
    wrap_graph(Graph::from_csr(n, std::move(off), std::move(tgt), keep_loops ? LoopPolicy::Keep : LoopPolicy::Ignore),
               out);
  });
}

lr_status lr_graph_load_edge_list(const char* path, int dense_ids, int keep_loops, lr_graph** out) {
  *out = nullptr;
  return guarded([&] {
    wrap_graph(load_edge_list(path, dense_ids != 0, keep_loops ? LoopPolicy::Keep : LoopPolicy::Ignore), out);
  });
}

lr_status lr_graph_parse_edge_buffer(const char* data, int64_t len, int dense_ids, int keep_loops, lr_graph** out) {
  *out = nullptr;
  return guarded([&] {
    if (len < 0 || (len > 0 && !data)) throw std::invalid_argument("bad buffer");
    wrap_graph(parse_edge_buffer(data, static_cast<std::size_t>(len), dense_ids != 0,
                                 keep_loops ? LoopPolicy::Keep : LoopPolicy::Ignore),
               out);
  });
}

int32_t lr_graph_vertex_count(const lr_graph* g) { return g ? g->g.vertex_count() : 0; }
int64_t lr_graph_edge_count(const lr_graph* g) { return g ? g->g.edge_count() : 0; }

lr_status lr_graph_csr(const lr_graph* gp, int64_t* offsets, int32_t* targets, uint8_t* has_loop, int32_t* walk_deg) {
  if (!gp) {
    lrerr::set("null graph");
    return LR_EINVAL;
  }
  const Graph& g = gp->g;
  const std::size_t n = static_cast<std::size_t>(g.vertex_count());
  if (offsets) std::memcpy(offsets, g.offsets_data(), (n + 1) * sizeof(int64_t));
  if (targets) std::memcpy(targets, g.targets_data(), static_cast<std::size_t>(g.edge_count()) * sizeof(int32_t));
  if (has_loop) std::memcpy(has_loop, g.loop_data(), n);
  if (walk_deg)
    for (VertexId u = 0; u < g.vertex_count(); ++u) walk_deg[u] = g.walk_out_degree(u);
  return LR_OK;
}

void lr_graph_free(lr_graph* g) { delete g; }

lr_status lr_find_components(const lr_graph* gp, int merge_cacs, int32_t* comp_of, int32_t* kinds, int32_t* levels,
                             int32_t* sizes, int32_t* k_out, int32_t* max_level, int64_t* stats3) {
  if (!gp) {
    lrerr::set("null graph");
    return LR_EINVAL;
  }
  return guarded([&] {
    PartitionStats st;
    const Partition p = merge_cacs ? find_components(gp->g, &st) : find_components_scc_only(gp->g);
    std::memcpy(comp_of, p.comp_of.data(), p.comp_of.size() * sizeof(int32_t));
    for (std::size_t c = 0; c < p.component_count(); ++c) {
      kinds[c] = p.kinds[c] == ComponentKind::Scc ? 0 : 1;
      levels[c] = p.levels[c];
      sizes[c] = p.sizes[c];
    }
    *k_out = static_cast<int32_t>(p.component_count());
    *max_level = p.max_level;
    if (stats3) {
      stats3[0] = merge_cacs ? st.explore_edge_visits : 0;
      stats3[1] = merge_cacs ? st.merge_scan_edge_visits : 0;
      stats3[2] = merge_cacs ? st.finish_calls : 0;
    }
  });
}

lr_status lr_plan_build(const lr_graph* gp, int32_t small_threshold, lr_plan** out) {
  *out = nullptr;
  if (!gp) {
    lrerr::set("null graph");
    return LR_EINVAL;
  }
  return guarded([&] {
    if (small_threshold < 1) throw std::invalid_argument("small_threshold must be at least 1");
    auto plan = std::make_unique<lr_plan>();
    plan->g = &gp->g;
    plan->threshold = small_threshold;
    if (std::getenv("LR_PLAN_PLAIN") != nullptr) {
      // the public two-call path (own transpose in the layout, every edge's
      // components looked up): what tests compare the shared-in-edge path with
      plan->p = find_components(gp->g);
      plan->L = build_layout(gp->g, plan->p, small_threshold);
    } else {
      detail::InEdges in;
      plan->p = detail::find_components_with_in_edges(gp->g, nullptr, in);
      plan->L = detail::build_layout_from(gp->g, plan->p, small_threshold, in);
    }
    *out = plan.release();
  });
}

void lr_plan_free(lr_plan* p) { delete p; }

lr_status lr_plan_build_baseline(const lr_graph* gp, lr_plan** out) {
  *out = nullptr;
  if (!gp) {
    lrerr::set("null graph");
    return LR_EINVAL;
  }
  return guarded([&] {
    auto plan = std::make_unique<lr_plan>();
    plan->g = &gp->g;
    plan->baseline = true;
    plan->L = build_baseline_layout(gp->g);
    *out = plan.release();
  });
}

static const Schedule& plan_schedule(lr_plan* p) {
  if (p->baseline) throw std::invalid_argument("a baseline plan has no schedule");
  if (!p->sched) p->sched = std::make_unique<Schedule>(build_schedule(*p->g, p->p, p->threshold));
  return *p->sched;
}

lr_status lr_plan_schedule_sizes(const lr_plan* cp, int64_t* o) {
  return guarded([&] {
    const Schedule& s = plan_schedule(const_cast<lr_plan*>(cp));
    int64_t units = 0, ids = 0, edges = 0, cross = 0;
    for (const auto& L : s.levels) {
      units += static_cast<int64_t>(L.units.size());
      for (const auto& u : L.units) {
        ids += u.size();
        edges += static_cast<int64_t>(u.edges.size());
      }
      cross += static_cast<int64_t>(L.cross_edges.size());
    }
    o[0] = static_cast<int64_t>(s.levels.size());
    o[1] = units;
    o[2] = ids;
    o[3] = edges;
    o[4] = cross;
    o[5] = s.intra_edge_count;
    o[6] = s.cross_edge_count;
    o[7] = s.dropped_loop_count;
  });
}

lr_status lr_plan_schedule_get(const lr_plan* cp, int32_t* level_values, int32_t* level_unit_begin,
                               int64_t* level_cross_begin, int32_t* unit_kind, int32_t* unit_level, int32_t* unit_size,
                               int64_t* unit_ids_begin, int64_t* unit_edges_begin, int32_t* ids, int32_t* edge_src,
                               int32_t* edge_dst, int32_t* cross_src, int32_t* cross_dst, int32_t* cross_deg,
                               int32_t* permutation) {
  return guarded([&] {
    const Schedule& s = plan_schedule(const_cast<lr_plan*>(cp));
    int64_t u = 0, id = 0, e = 0, x = 0;
    for (std::size_t li = 0; li < s.levels.size(); ++li) {
      const auto& L = s.levels[li];
      level_values[li] = L.level;
      level_unit_begin[li] = static_cast<int32_t>(u);
      level_cross_begin[li] = x;
      for (const auto& un : L.units) {
        unit_kind[u] = static_cast<int32_t>(un.kind);
        unit_level[u] = un.level;
        unit_size[u] = un.size();
        unit_ids_begin[u] = id;
        unit_edges_begin[u] = e;
        for (const VertexId v : un.global_ids) ids[id++] = v;
        for (const auto& [a, b] : un.edges) {
          edge_src[e] = a;
          edge_dst[e] = b;
          ++e;
        }
        ++u;
      }
      for (const auto& ce : L.cross_edges) {
        cross_src[x] = ce.src;
        cross_dst[x] = ce.dst;
        cross_deg[x] = ce.src_out_degree;
        ++x;
      }
    }
    level_unit_begin[s.levels.size()] = static_cast<int32_t>(u);
    level_cross_begin[s.levels.size()] = x;
    unit_ids_begin[u] = id;
    unit_edges_begin[u] = e;
    std::memcpy(permutation, s.permutation.data(), s.permutation.size() * sizeof(int32_t));
  });
}

lr_status lr_plan_census(const lr_plan* p, lr_census* out) {
  return guarded([&] {
    if (p->baseline) throw std::invalid_argument("a baseline plan has no partition");
    const PartitionCensus c = census(p->p);
    out->components = c.components;
    out->scc_components = c.scc_components;
    out->cac_components = c.cac_components;
    out->singleton_cacs = c.singleton_cacs;
    out->largest_component = c.largest_component;
    out->largest_is_scc = c.largest_kind == ComponentKind::Scc;
    out->max_level = c.max_level;
    out->level_count = c.level_count;
  });
}

lr_status lr_plan_layout(const lr_plan* p, lr_layout* o) {
  if (!p || !o) {
    lrerr::set("null plan");
    return LR_EINVAL;
  }
  const Layout& L = p->L;
  o->n = L.n;
  o->n_levels = L.level_count();
  o->keep_loops = L.keep_loops;
  o->n_units = L.unit_count();
  o->nnz_cross = static_cast<int64_t>(L.xsrc.size());
  o->nnz_intra = static_cast<int64_t>(L.isrc.size());
  o->depth_ptr_len = static_cast<int64_t>(L.depth_ptr.size());
  o->level_row_begin = L.level_row_begin.data();
  o->level_unit_begin = L.level_unit_begin.data();
  o->vertex_of = L.vertex_of.data();
  o->row_of = L.row_of.data();
  o->deg = L.deg.data();
  o->loop = L.loop.data();
  o->xptr = L.xptr.data();
  o->xsrc = L.xsrc.data();
  o->iptr = L.iptr.data();
  o->isrc = L.isrc.data();
  o->unit_kind = L.unit_kind.data();
  o->unit_level = L.unit_level.data();
  o->unit_row_begin = L.unit_row_begin.data();
  o->unit_edges = L.unit_edges.data();
  o->cac_depth_begin = L.cac_depth_begin.data();
  o->depth_ptr = L.depth_ptr.data();
  return LR_OK;
}

lr_status lr_validate_params(double c, double tol) {
  if (!(c > 0.0) || !(c < 1.0)) {
    lrerr::set("continuation probability must lie in (0, 1)");
    return LR_EINVAL;
  }
  if (!(tol > 0.0)) {
    lrerr::set("tolerance must be positive");
    return LR_EINVAL;
  }
  return LR_OK;
}

int64_t lr_iteration_cap(double c, double tol) {
  const double steps = std::log(tol) / std::log(c);
  const double capped = 10.0 * std::ceil(std::max(1.0, steps));
  return std::max<int64_t>(static_cast<int64_t>(capped), 16);
}

void lr_error_bound(int64_t large, int64_t n, double c, double tol, double* out2) {
  out2[0] = static_cast<double>(large) * tol * c / (1.0 - c);
  out2[1] = n > 0 ? out2[0] / static_cast<double>(n) : 0.0;
}

lr_status lr_compute_pagerank(const lr_graph* gp, const double* w, int64_t wn, double c, double tol,
                              int32_t small_threshold, int device, double* ranks, double* r1, lr_report* rep,
                              int64_t* unit_iters, int64_t unit_cap) {
  if (!gp) {
    lrerr::set("null graph");
    return LR_EINVAL;
  }
  lr_status st = lr_validate_params(c, tol);
  if (st != LR_OK) return st;
  const Graph& g = gp->g;
  const int64_t n = g.vertex_count();
  if (wn != n) {
    lrerr::set("weight vector does not match the vertex count");
    return LR_EINVAL;
  }
  for (int64_t v = 0; v < n; ++v)
    if (w[v] < 0.0) {
      lrerr::set("weights must be non-negative");
      return LR_EINVAL;
    }
  const auto t0 = std::chrono::steady_clock::now();
  lr_report local{};
  if (!rep) rep = &local;
  std::memset(rep, 0, sizeof *rep);
  rep->vertices = n;
  rep->edges = g.edge_count();
  rep->max_level = -1;
  rep->threads = 1;
  if (n == 0) return LR_OK;
  double wmax = w[0];
  for (int64_t v = 1; v < n; ++v) wmax = std::max(wmax, w[v]);
  rep->all_weights_zero = wmax == 0.0;

  lr_plan* plan = nullptr;
  st = lr_plan_build(gp, small_threshold, &plan);
  if (st != LR_OK) return st;
  std::unique_ptr<lr_plan, void (*)(lr_plan*)> plan_guard(plan, lr_plan_free);
  rep->plan_ms = ms_since(t0);
  lr_census cs{};
  lr_plan_census(plan, &cs);
  rep->components = cs.components;
  rep->scc_components = cs.scc_components;
  rep->cac_components = cs.cac_components;
  rep->singleton_cacs = cs.singleton_cacs;
  rep->largest_component = cs.largest_component;
  rep->largest_is_scc = cs.largest_is_scc;
  rep->max_level = cs.max_level;
  rep->level_count = cs.level_count;

  lr_ctx* ctx = nullptr;
  st = lr_ctx_create(device, &ctx);
  if (st != LR_OK) return st;
  std::unique_ptr<lr_ctx, void (*)(lr_ctx*)> ctx_guard(ctx, lr_ctx_free);
  lr_layout lay{};
  lr_plan_layout(plan, &lay);
  const auto t1 = std::chrono::steady_clock::now();
  st = lr_ctx_upload(ctx, &lay);
  if (st != LR_OK) return st;
  rep->upload_ms = ms_since(t1);
  std::vector<int64_t> iters(static_cast<std::size_t>(lay.n_units), 0);
  lr_solve_info info{};
  const auto t2 = std::chrono::steady_clock::now();
  st = lr_solve(ctx, w, c, tol, ranks, r1, &info, iters.data());
  rep->solve_ms = ms_since(t2);
  rep->device_ms = info.device_ms;
  if (st != LR_OK) return st;

  const Layout& L = plan->L;
  rep->n_units = L.unit_count();
  rep->cross_edge_count = L.cross_edge_count;
  for (int64_t u = 0; u < L.unit_count(); ++u) {
    const std::size_t su = static_cast<std::size_t>(u);
    const int64_t it = iters[su];
    const int64_t e = L.unit_edges[su];
    const int64_t size = L.unit_row_begin[su + 1] - L.unit_row_begin[su];
    rep->total_iterations += it;
    if (L.unit_kind[su] == static_cast<std::uint8_t>(UnitKind::SccLarge)) {
      rep->iterative_edge_work += it * e;
      rep->iterative_edges += e;
      rep->large_scc_vertices += size;
    } else {
      rep->single_pass_edge_work += e;
    }
    if (unit_iters && u < unit_cap) unit_iters[u] = it;
  }
  rep->single_pass_edge_work += L.cross_edge_count;
  rep->total_edge_work = rep->iterative_edge_work + rep->single_pass_edge_work;
  rep->mean_iterations_per_edge =
      rep->iterative_edges > 0 ? static_cast<double>(rep->iterative_edge_work) / static_cast<double>(rep->iterative_edges)
                               : 0.0;
  double eb[2];
  lr_error_bound(rep->large_scc_vertices, n, c, tol, eb);
  rep->eps_tot = eb[0];
  rep->eps_avg = eb[1];
  rep->wall_ms = ms_since(t0);
  return LR_OK;
}

}  // extern "C"

namespace levelrank {
inline namespace b200 {
namespace detail {
// compute_baseline on a C++ Graph (the C-ABI entry and the C++ API both land here)
lr_status baseline_solve(const Graph& g, const double* w, int64_t wn, double c, double tol, int device, double* ranks,
                         double* r1, lr_report* rep) {
  lr_status st = lr_validate_params(c, tol);
  if (st != LR_OK) return st;
  const int64_t n = g.vertex_count();
  if (wn != n) {
    lrerr::set("weight vector does not match the vertex count");
    return LR_EINVAL;
  }
  for (int64_t v = 0; v < n; ++v)
    if (w[v] < 0.0) {
      lrerr::set("weights must be non-negative");
      return LR_EINVAL;
    }
  const auto t0 = std::chrono::steady_clock::now();
  lr_report local{};
  if (!rep) rep = &local;
  std::memset(rep, 0, sizeof *rep);
  rep->vertices = n;
  rep->edges = g.edge_count();
  rep->max_level = -1;
  rep->threads = 1;
  if (n == 0) return LR_OK;
  double wmax = w[0];
  for (int64_t v = 1; v < n; ++v) wmax = std::max(wmax, w[v]);
  rep->all_weights_zero = wmax == 0.0;
  std::unique_ptr<lr_plan> plan;
  st = guarded([&] {
    plan = std::make_unique<lr_plan>();
    plan->g = &g;
    plan->baseline = true;
    plan->L = build_baseline_layout(g);
  });
  if (st != LR_OK) return st;
  rep->plan_ms = ms_since(t0);
  lr_ctx* ctx = nullptr;
  st = lr_ctx_create(device, &ctx);
  if (st != LR_OK) return st;
  std::unique_ptr<lr_ctx, void (*)(lr_ctx*)> ctx_guard(ctx, lr_ctx_free);
  lr_layout lay{};
  lr_plan_layout(plan.get(), &lay);
  const auto t1 = std::chrono::steady_clock::now();
  st = lr_ctx_upload(ctx, &lay);
  if (st != LR_OK) return st;
  rep->upload_ms = ms_since(t1);
  int64_t iters = 0;
  lr_solve_info info{};
  const auto t2 = std::chrono::steady_clock::now();
  st = lr_solve(ctx, w, c, tol, ranks, r1, &info, &iters);
  rep->solve_ms = ms_since(t2);
  rep->device_ms = info.device_ms;
  if (st != LR_OK) return st;
  // engine.cpp:210-215
  const int64_t walk_edges = plan->L.unit_edges[0];
  rep->n_units = 1;
  rep->total_iterations = iters;
  rep->iterative_edge_work = iters * walk_edges;
  rep->iterative_edges = walk_edges;
  rep->total_edge_work = rep->iterative_edge_work;
  rep->mean_iterations_per_edge = static_cast<double>(iters);
  rep->wall_ms = ms_since(t0);
  return LR_OK;
}
}  // namespace detail
}  // namespace b200
}  // namespace levelrank

extern "C" {

lr_status lr_compute_baseline(const lr_graph* gp, const double* w, int64_t wn, double c, double tol, int device,
                              double* ranks, double* r1, lr_report* rep) {
  if (!gp) {
    lrerr::set("null graph");
    return LR_EINVAL;
  }
  return levelrank::detail::baseline_solve(gp->g, w, wn, c, tol, device, ranks, r1, rep);
}

lr_status lr_gen_rmat(int32_t scale, int64_t edge_factor, double a, double b, double c, uint64_t seed, lr_graph** out) {
  *out = nullptr;
  return guarded([&] { wrap_graph(gen::rmat(scale, edge_factor, a, b, c, seed), out); });
}

lr_status lr_graph_dangle(const lr_graph* g, double p, uint64_t seed, lr_graph** out) {
  *out = nullptr;
  if (!g) {
    lrerr::set("null graph");
    return LR_EINVAL;
  }
  return guarded([&] { wrap_graph(gen::dangle(g->g, p, seed), out); });
}

lr_status lr_gen_planted(int32_t n, int32_t n_scc, int32_t scc_min, int32_t scc_max, int64_t budget, double out_degree,
                         int64_t inter_edges, double dangling_fraction, uint64_t seed, lr_graph** out) {
  *out = nullptr;
  return guarded([&] {
    wrap_graph(gen::planted(n, n_scc, scc_min, scc_max, budget, out_degree, inter_edges, dangling_fraction, seed), out);
  });
}

lr_status lr_gen_deep_dag(int32_t levels, int32_t width, int32_t scc_min, int32_t scc_max, double scc_out_degree,
                          int32_t branch_min, int32_t branch_max, double inter_out_degree, int32_t reach, uint64_t seed,
                          lr_graph** out) {
  *out = nullptr;
  return guarded([&] {
    wrap_graph(gen::deep_dag(levels, width, scc_min, scc_max, scc_out_degree, branch_min, branch_max, inter_out_degree,
                             reach, seed),
               out);
  });
}

}  // extern "C"

// ------------------------------------------------------------ output formats
namespace {
lr_status emit(const std::string& text, char** out, int64_t* len) {
  char* buf = static_cast<char*>(std::malloc(text.size() + 1));
  if (!buf) {
    lrerr::set("out of host memory");
    return LR_ENOMEM;
  }
  std::memcpy(buf, text.data(), text.size());
  buf[text.size()] = '\0';
  *out = buf;
  if (len) *len = static_cast<int64_t>(text.size());
  return LR_OK;
}
}  // namespace

extern "C" {

lr_status lr_report_format(const lr_report* r, const lr_report_meta* meta, const lr_unit_record* units,
                           int64_t n_units, int fmt, char** out, int64_t* len) {
  if (!out || (fmt != 3 && (!r || !meta)) || n_units < 0 || (n_units > 0 && !units) || fmt < 0 || fmt > 3) {
    lrerr::set("bad report format request");
    return LR_EINVAL;
  }
  *out = nullptr;
  std::ostringstream os;
  lr_status st = guarded([&] {
    if (fmt == 3) {
      write_bench_header(os);
      return;
    }
    SolveReport rep;
    rep.method = meta->method ? meta->method : "partitioned";
    rep.mode = meta->mode ? meta->mode : "sequential";
    rep.c = meta->c;
    rep.tol = meta->tol;
    rep.keep_loops = meta->keep_loops != 0;
    rep.small_threshold = meta->small_threshold;
    rep.threads = meta->threads;
    rep.vertices = r->vertices;
    rep.edges = r->edges;
    rep.components = r->components;
    rep.scc_components = r->scc_components;
    rep.cac_components = r->cac_components;
    rep.singleton_cacs = r->singleton_cacs;
    rep.largest_component = r->largest_component;
    rep.largest_component_kind = r->largest_is_scc ? "scc" : "cac";
    rep.max_level = r->max_level;
    rep.level_count = r->level_count;
    rep.large_scc_vertices = r->large_scc_vertices;
    rep.eps_tot = r->eps_tot;
    rep.eps_avg = r->eps_avg;
    rep.total_iterations = r->total_iterations;
    rep.iterative_edge_work = r->iterative_edge_work;
    rep.iterative_edges = r->iterative_edges;
    rep.single_pass_edge_work = r->single_pass_edge_work;
    rep.cross_edge_count = r->cross_edge_count;
    rep.total_edge_work = r->total_edge_work;
    rep.mean_iterations_per_edge = r->mean_iterations_per_edge;
    rep.all_weights_zero = r->all_weights_zero != 0;
    rep.wall_ms = r->wall_ms;
    rep.units.resize(static_cast<std::size_t>(n_units));
    for (int64_t i = 0; i < n_units; ++i) {
      const lr_unit_record& u = units[i];
      rep.units[static_cast<std::size_t>(i)] =
          UnitRecord{static_cast<UnitKind>(u.kind), u.level, u.size, u.edges, u.iterations, u.wall_ms};
    }
    if (fmt == 0) rep.write_text(os);
    else if (fmt == 1) rep.write_json(os);
    else write_bench_row(os, rep);
  });
  if (st != LR_OK) return st;
  return emit(os.str(), out, len);
}

lr_status lr_ranks_format(const double* ranks, int64_t n, char** out, int64_t* len) {
  if (!out || n < 0 || (n > 0 && !ranks)) {
    lrerr::set("bad ranks");
    return LR_EINVAL;
  }
  *out = nullptr;
  std::ostringstream os;
  lr_status st = guarded([&] { write_ranks(os, std::span<const double>(ranks, static_cast<std::size_t>(n))); });
  if (st != LR_OK) return st;
  return emit(os.str(), out, len);
}

lr_status lr_ranks_write(const double* ranks, int64_t n, const char* path) {
  if (!path || n < 0 || (n > 0 && !ranks)) {
    lrerr::set("bad ranks");
    return LR_EINVAL;
  }
  return guarded([&] {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw IoError(std::string("cannot open ") + path + " for writing");
    write_ranks(f, std::span<const double>(ranks, static_cast<std::size_t>(n)));
    f.flush();
    if (!f) throw IoError(std::string("write to ") + path + " failed");
  });
}

void lr_string_free(char* s) { std::free(s); }

}  // extern "C"

extern "C" lr_status lr_solve_unit(const lr_graph* g, int kind, const int32_t* global_ids, int32_t m,
                                   const int32_t* edge_src, const int32_t* edge_dst, int64_t n_edges,
                                   const double* w_local, double c, double tol, int device, double* ranks_out,
                                   int64_t* iterations_out, int64_t* edge_visits_out) {
  if (!g || m < 0 || n_edges < 0 || (m > 0 && (!global_ids || !w_local || !ranks_out)) ||
      (n_edges > 0 && (!edge_src || !edge_dst)) || kind < 0 || kind > 3) {
    lrerr::set("bad unit solve request");
    return LR_EINVAL;
  }
  return guarded([&] {
    SolveUnit unit;
    unit.kind = static_cast<UnitKind>(kind);
    unit.global_ids.assign(global_ids, global_ids + m);
    unit.edges.resize(static_cast<std::size_t>(n_edges));
    for (int64_t i = 0; i < n_edges; ++i) unit.edges[static_cast<std::size_t>(i)] = {edge_src[i], edge_dst[i]};
    const std::span<const double> w(w_local, static_cast<std::size_t>(m));
    const SolverParams params{c, tol};
    std::vector<double> r;
    std::int64_t it = 0;
    EdgeId visits = 0;
    switch (kind) {
      case 0: r = solve_singletons(g->g, unit, w, params, device); break;
      case 1: r = solve_cac(g->g, unit, w, params, &visits, device); break;
      case 2: r = solve_small_scc(g->g, unit, w, params, device); break;
      default: r = solve_large_scc(g->g, unit, w, params, it, nullptr, device); break;
    }
    std::copy(r.begin(), r.end(), ranks_out);
    if (iterations_out) *iterations_out = it;
    if (edge_visits_out) *edge_visits_out = visits;
  });
}

extern "C" lr_status lr_solve_large_scc_stats(const lr_graph* g, const int32_t* global_ids, int32_t m,
                                              const int32_t* edge_src, const int32_t* edge_dst, int64_t n_edges,
                                              const double* w_local, double c, double tol, int device,
                                              double* ranks_out, int64_t* iterations_out, double* l1, int64_t l1_cap,
                                              int64_t* l1_len, double* min_entry) {
  if (!g || m < 0 || n_edges < 0 || (m > 0 && (!global_ids || !w_local || !ranks_out)) ||
      (n_edges > 0 && (!edge_src || !edge_dst)) || !iterations_out || !min_entry) {
    lrerr::set("bad unit solve request");
    return LR_EINVAL;
  }
  return guarded([&] {
    SolveUnit unit;
    unit.kind = UnitKind::SccLarge;
    unit.global_ids.assign(global_ids, global_ids + m);
    unit.edges.resize(static_cast<std::size_t>(n_edges));
    for (int64_t i = 0; i < n_edges; ++i) unit.edges[static_cast<std::size_t>(i)] = {edge_src[i], edge_dst[i]};
    PowerSeriesStats st;
    std::int64_t it = 0;
    const std::vector<double> r =
        solve_large_scc(g->g, unit, std::span<const double>(w_local, static_cast<std::size_t>(m)), SolverParams{c, tol},
                        it, &st, device);
    std::copy(r.begin(), r.end(), ranks_out);
    *iterations_out = it;
    const int64_t k = std::min<int64_t>(l1_cap, static_cast<int64_t>(st.increment_l1_norms.size()));
    if (l1) std::copy(st.increment_l1_norms.begin(), st.increment_l1_norms.begin() + k, l1);
    if (l1_len) *l1_len = static_cast<int64_t>(st.increment_l1_norms.size());
    *min_entry = st.min_increment_entry;
  });
}
