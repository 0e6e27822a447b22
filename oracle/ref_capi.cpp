// TEST INFRASTRUCTURE ONLY -- the checker, never the product.
//
// A thin extern "C" driver around the *unmodified* reference levelrank
// sources (compiled straight out of /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/).  It lets the Python tests and the
// bench's reference arm call the reference's own public API:
//   Graph::from_edges            proj/src/graph.cpp:14-36
//   parse_edge_list              proj/src/graph.cpp:54-99
//   find_components / _scc_only  proj/src/partition.cpp:246-250
//   build_schedule               proj/src/schedule.cpp:32-137
//   compute_pagerank             proj/src/engine.cpp:89-182
//   compute_baseline             proj/src/engine.cpp:184-218
//   oracle_r1_to_r3              proj/src/solvers.cpp:200-244
//   solve_dense_whole            proj/src/solvers.cpp:118-126
// plus a restated level loop (engine.cpp:126-158) that calls the
// reference's own unit solvers and propagate_weights, used by bench.py to
// time the reference CPU path on a prepared schedule.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <iomanip>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "levelrank/engine.hpp"
#include "levelrank/graph.hpp"
#include "levelrank/partition.hpp"
#include "levelrank/schedule.hpp"
#include "levelrank/solvers.hpp"

using namespace levelrank;

namespace {

thread_local std::string g_err;

int fail_from_current() {
  try {
    throw;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

Eigen::VectorXd to_vec(const double* p, std::int64_t n) {
  Eigen::VectorXd v(n);
  for (std::int64_t i = 0; i < n; ++i) v(i) = p[i];
  return v;
}

struct RefPartition {
  Partition p;
  PartitionStats stats;
};

struct FlatSchedule {
  Schedule s;
  // flattened unit view, level-major
  std::vector<std::int32_t> unit_kind, unit_level, unit_size;
  std::vector<std::int64_t> unit_ids_begin, unit_edges_begin;
  std::vector<std::int32_t> ids;
  std::vector<std::int32_t> edge_src, edge_dst;
  std::vector<std::int64_t> level_cross_begin;
  std::vector<std::int32_t> cross_src, cross_dst, cross_deg;
  std::vector<std::int32_t> level_values, level_unit_begin;
};

struct Prep {
  Partition p;
  Schedule s;
};

}  // namespace

extern "C" {

typedef struct {
  int64_t vertices, edges, components, scc_components, cac_components, singleton_cacs;
  int32_t largest_component, largest_is_scc, max_level, level_count;
  int64_t large_scc_vertices;
  double eps_tot, eps_avg;
  int64_t total_iterations, iterative_edge_work, iterative_edges, single_pass_edge_work,
      cross_edge_count, total_edge_work;
  double mean_iterations_per_edge;
  int32_t all_weights_zero, threads;
  double wall_ms;
  int64_t n_units;
} lrref_report;

const char* lrref_last_error(void) { return g_err.c_str(); }

void* lrref_graph_new(int32_t n, const int32_t* src, const int32_t* dst, int64_t m, int keep) {
  try {
    std::vector<std::pair<VertexId, VertexId>> e(static_cast<std::size_t>(m));
    for (int64_t i = 0; i < m; ++i) e[static_cast<std::size_t>(i)] = {src[i], dst[i]};
    return new Graph(Graph::from_edges(n, std::move(e), keep ? LoopPolicy::Keep : LoopPolicy::Ignore));
  } catch (...) {
    fail_from_current();
    return nullptr;
  }
}
// parse_edge_list (proj/src/graph.cpp:54-99) on a byte buffer; NULL and the
// exception message in lrref_last_error() on failure.
void* lrref_graph_parse(const char* data, int64_t len, int dense_ids) {
  try {
    std::istringstream in(std::string(data, static_cast<std::size_t>(len)));
    return new Graph(parse_edge_list(in, dense_ids != 0));
  } catch (...) {
    fail_from_current();
    return nullptr;
  }
}
void lrref_graph_free(void* g) { delete static_cast<Graph*>(g); }
int64_t lrref_graph_edge_count(void* g) { return static_cast<Graph*>(g)->edge_count(); }
int32_t lrref_graph_vertex_count(void* g) { return static_cast<Graph*>(g)->vertex_count(); }
void lrref_graph_csr(void* gp, int64_t* offsets, int32_t* targets, uint8_t* has_loop,
                     int32_t* walk_deg) {
  const Graph& g = *static_cast<Graph*>(gp);
  offsets[0] = 0;
  int64_t k = 0;
  for (VertexId u = 0; u < g.vertex_count(); ++u) {
    for (VertexId v : g.out_neighbors(u)) targets[k++] = v;
    offsets[u + 1] = k;
    has_loop[u] = g.has_loop(u) ? 1 : 0;
    walk_deg[u] = g.walk_out_degree(u);
  }
}

// mode 0: find_components, 1: find_components_scc_only, 2: reference_partition
void* lrref_partition_new(void* gp, int mode) {
  try {
    const Graph& g = *static_cast<Graph*>(gp);
    auto* rp = new RefPartition;
    if (mode == 0)
      rp->p = find_components(g, &rp->stats);
    else if (mode == 1)
      rp->p = find_components_scc_only(g);
    else
      rp->p = reference_partition(g);
    return rp;
  } catch (...) {
    fail_from_current();
    return nullptr;
  }
}
void lrref_partition_free(void* p) { delete static_cast<RefPartition*>(p); }
int64_t lrref_partition_count(void* p) {
  return static_cast<int64_t>(static_cast<RefPartition*>(p)->p.component_count());
}
void lrref_partition_get(void* pp, int32_t* comp_of, int32_t* kinds, int32_t* levels,
                         int32_t* sizes, int32_t* max_level, int64_t* stats3) {
  const RefPartition& rp = *static_cast<RefPartition*>(pp);
  const Partition& p = rp.p;
  for (std::size_t v = 0; v < p.comp_of.size(); ++v) comp_of[v] = p.comp_of[v];
  for (std::size_t c = 0; c < p.kinds.size(); ++c) {
    kinds[c] = p.kinds[c] == ComponentKind::Scc ? 0 : 1;
    levels[c] = p.levels[c];
    sizes[c] = p.sizes[c];
  }
  *max_level = p.max_level;
  if (stats3) {
    stats3[0] = rp.stats.explore_edge_visits;
    stats3[1] = rp.stats.merge_scan_edge_visits;
    stats3[2] = rp.stats.finish_calls;
  }
}
int lrref_validate_partition(void* gp, void* pp) {
  return static_cast<int>(
      validate_partition(*static_cast<Graph*>(gp), static_cast<RefPartition*>(pp)->p).size());
}

void* lrref_schedule_new(void* gp, void* pp, int32_t threshold) {
  try {
    const Graph& g = *static_cast<Graph*>(gp);
    auto* fs = new FlatSchedule;
    fs->s = build_schedule(g, static_cast<RefPartition*>(pp)->p, threshold);
    for (const auto& L : fs->s.levels) {
      fs->level_values.push_back(L.level);
      fs->level_unit_begin.push_back(static_cast<int32_t>(fs->unit_kind.size()));
      fs->level_cross_begin.push_back(static_cast<int64_t>(fs->cross_src.size()));
      for (const auto& u : L.units) {
        fs->unit_kind.push_back(static_cast<int32_t>(u.kind));
        fs->unit_level.push_back(u.level);
        fs->unit_size.push_back(u.size());
        fs->unit_ids_begin.push_back(static_cast<int64_t>(fs->ids.size()));
        fs->unit_edges_begin.push_back(static_cast<int64_t>(fs->edge_src.size()));
        for (auto v : u.global_ids) fs->ids.push_back(v);
        for (auto [a, b] : u.edges) {
          fs->edge_src.push_back(a);
          fs->edge_dst.push_back(b);
        }
      }
      for (const auto& e : L.cross_edges) {
        fs->cross_src.push_back(e.src);
        fs->cross_dst.push_back(e.dst);
        fs->cross_deg.push_back(e.src_out_degree);
      }
    }
    fs->level_unit_begin.push_back(static_cast<int32_t>(fs->unit_kind.size()));
    fs->level_cross_begin.push_back(static_cast<int64_t>(fs->cross_src.size()));
    fs->unit_ids_begin.push_back(static_cast<int64_t>(fs->ids.size()));
    fs->unit_edges_begin.push_back(static_cast<int64_t>(fs->edge_src.size()));
    return fs;
  } catch (...) {
    fail_from_current();
    return nullptr;
  }
}
void lrref_schedule_free(void* s) { delete static_cast<FlatSchedule*>(s); }
// sizes: [n_levels, n_units, n_ids, n_edges, n_cross, intra, cross, dropped]
void lrref_schedule_sizes(void* sp, int64_t* out8) {
  const FlatSchedule& fs = *static_cast<FlatSchedule*>(sp);
  out8[0] = static_cast<int64_t>(fs.level_values.size());
  out8[1] = static_cast<int64_t>(fs.unit_kind.size());
  out8[2] = static_cast<int64_t>(fs.ids.size());
  out8[3] = static_cast<int64_t>(fs.edge_src.size());
  out8[4] = static_cast<int64_t>(fs.cross_src.size());
  out8[5] = fs.s.intra_edge_count;
  out8[6] = fs.s.cross_edge_count;
  out8[7] = fs.s.dropped_loop_count;
}
void lrref_schedule_get(void* sp, int32_t* level_values, int32_t* level_unit_begin,
                        int64_t* level_cross_begin, int32_t* unit_kind, int32_t* unit_level,
                        int32_t* unit_size, int64_t* unit_ids_begin, int64_t* unit_edges_begin,
                        int32_t* ids, int32_t* edge_src, int32_t* edge_dst, int32_t* cross_src,
                        int32_t* cross_dst, int32_t* cross_deg, int32_t* permutation) {
  const FlatSchedule& fs = *static_cast<FlatSchedule*>(sp);
  auto cp32 = [](int32_t* dst, const std::vector<int32_t>& v) {
    if (!v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(int32_t));
  };
  auto cp64 = [](int64_t* dst, const std::vector<int64_t>& v) {
    if (!v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(int64_t));
  };
  cp32(level_values, fs.level_values);
  cp32(level_unit_begin, fs.level_unit_begin);
  cp64(level_cross_begin, fs.level_cross_begin);
  cp32(unit_kind, fs.unit_kind);
  cp32(unit_level, fs.unit_level);
  cp32(unit_size, fs.unit_size);
  cp64(unit_ids_begin, fs.unit_ids_begin);
  cp64(unit_edges_begin, fs.unit_edges_begin);
  cp32(ids, fs.ids);
  cp32(edge_src, fs.edge_src);
  cp32(edge_dst, fs.edge_dst);
  cp32(cross_src, fs.cross_src);
  cp32(cross_dst, fs.cross_dst);
  cp32(cross_deg, fs.cross_deg);
  for (std::size_t v = 0; v < fs.s.permutation.size(); ++v) permutation[v] = fs.s.permutation[v];
}

static void fill_report(const SolveReport& r, lrref_report* out) {
  out->vertices = r.vertices;
  out->edges = r.edges;
  out->components = r.components;
  out->scc_components = r.scc_components;
  out->cac_components = r.cac_components;
  out->singleton_cacs = r.singleton_cacs;
  out->largest_component = r.largest_component;
  out->largest_is_scc = r.largest_component_kind == "scc";
  out->max_level = r.max_level;
  out->level_count = r.level_count;
  out->large_scc_vertices = r.large_scc_vertices;
  out->eps_tot = r.eps_tot;
  out->eps_avg = r.eps_avg;
  out->total_iterations = r.total_iterations;
  out->iterative_edge_work = r.iterative_edge_work;
  out->iterative_edges = r.iterative_edges;
  out->single_pass_edge_work = r.single_pass_edge_work;
  out->cross_edge_count = r.cross_edge_count;
  out->total_edge_work = r.total_edge_work;
  out->mean_iterations_per_edge = r.mean_iterations_per_edge;
  out->all_weights_zero = r.all_weights_zero;
  out->threads = r.threads;
  out->wall_ms = r.wall_ms;
  out->n_units = static_cast<int64_t>(r.units.size());
}

// unit_iters (optional, size >= number of units): per-unit iteration counts in
// schedule order; unit_kinds likewise.
int lrref_compute_pagerank(void* gp, const double* w, int64_t wn, double c, double tol,
                           int parallel, int32_t threshold, int threads, double* ranks_out,
                           lrref_report* rep, int64_t* unit_iters, int32_t* unit_kinds,
                           int64_t unit_cap) {
  try {
    const Graph& g = *static_cast<Graph*>(gp);
    const auto res = compute_pagerank(g, to_vec(w, wn), SolverParams{c, tol},
                                      parallel ? ExecutionMode::Parallel : ExecutionMode::Sequential,
                                      threshold, threads);
    for (int64_t i = 0; i < res.ranks.size(); ++i) ranks_out[i] = res.ranks(i);
    if (rep) fill_report(res.report, rep);
    if (unit_iters)
      for (std::size_t u = 0; u < res.report.units.size() && static_cast<int64_t>(u) < unit_cap; ++u) {
        unit_iters[u] = res.report.units[u].iterations;
        if (unit_kinds) unit_kinds[u] = static_cast<int32_t>(res.report.units[u].kind);
      }
    return 0;
  } catch (...) {
    return fail_from_current();
  }
}

int lrref_compute_baseline(void* gp, const double* w, int64_t wn, double c, double tol,
                           double* ranks_out, lrref_report* rep) {
  try {
    const Graph& g = *static_cast<Graph*>(gp);
    const auto res = compute_baseline(g, to_vec(w, wn), SolverParams{c, tol});
    for (int64_t i = 0; i < res.ranks.size(); ++i) ranks_out[i] = res.ranks(i);
    if (rep) fill_report(res.report, rep);
    return 0;
  } catch (...) {
    return fail_from_current();
  }
}

int lrref_oracle_bridge(void* gp, const double* w, int64_t wn, double c, double* r1, double* r3,
                        double* d) {
  try {
    const auto b = oracle_r1_to_r3(*static_cast<Graph*>(gp), to_vec(w, wn), c);
    for (int64_t i = 0; i < b.r1.size(); ++i) {
      r1[i] = b.r1(i);
      r3[i] = b.r3(i);
    }
    *d = b.d;
    return 0;
  } catch (...) {
    return fail_from_current();
  }
}

int lrref_dense_whole(void* gp, const double* w, int64_t wn, double c, double* out) {
  try {
    const auto r = solve_dense_whole(*static_cast<Graph*>(gp), to_vec(w, wn), c);
    for (int64_t i = 0; i < r.size(); ++i) out[i] = r(i);
    return 0;
  } catch (...) {
    return fail_from_current();
  }
}

int64_t lrref_iteration_cap(double c, double tol) { return iteration_cap(SolverParams{c, tol}); }

void lrref_error_bound(int64_t large, int64_t n, double c, double tol, double* out2) {
  const auto b = error_bound(large, n, SolverParams{c, tol});
  out2[0] = b.eps_tot;
  out2[1] = b.eps_avg;
}

void lrref_propagate(const int32_t* src, const int32_t* dst, const int32_t* deg, int64_t m,
                     const double* ranks, int64_t n, double c, double* weights_inout) {
  std::vector<CrossEdge> cross(static_cast<std::size_t>(m));
  for (int64_t i = 0; i < m; ++i) cross[static_cast<std::size_t>(i)] = {src[i], dst[i], deg[i]};
  Eigen::VectorXd r = to_vec(ranks, n);
  Eigen::VectorXd w = to_vec(weights_inout, n);
  propagate_weights(cross, r, c, w);
  for (int64_t i = 0; i < n; ++i) weights_inout[i] = w(i);
}

// ---- bench reference arm: partition + schedule once, then time the level loop.
void* lrref_prep_new(void* gp, int32_t threshold) {
  try {
    const Graph& g = *static_cast<Graph*>(gp);
    auto* p = new Prep;
    p->p = find_components(g);
    p->s = build_schedule(g, p->p, threshold);
    return p;
  } catch (...) {
    fail_from_current();
    return nullptr;
  }
}
void lrref_prep_free(void* p) { delete static_cast<Prep*>(p); }

// The level loop of compute_pagerank (engine.cpp:126-158) over the prepared
// schedule, calling the reference's own unit solvers and propagate_weights.
// large_tol > 0 replaces tol for SccLarge units only (a bounded sample of the
// power series); large_tol <= 0 keeps the real tolerance.  Returns the edge
// work actually performed (same accounting as engine.cpp:160-172).
int lrref_prep_solve(void* gp, void* pp, const double* w, int64_t wn, double c, double tol,
                     double large_tol, int threads, double* ranks_out, int64_t* edge_work_out,
                     int64_t* large_iters_out, double* ms_out) {
  try {
    const Graph& g = *static_cast<Graph*>(gp);
    const Prep& prep = *static_cast<Prep*>(pp);
    const SolverParams params{c, tol};
    const SolverParams large_params{c, large_tol > 0 ? large_tol : tol};
    const auto t0 = std::chrono::steady_clock::now();
    Eigen::VectorXd work_w = to_vec(w, wn);
    Eigen::VectorXd ranks = Eigen::VectorXd::Zero(wn);
    std::atomic<int64_t> work{0}, iters{0};
    auto solve_one = [&](const SolveUnit& unit) {
      Eigen::VectorXd wl(unit.size());
      for (VertexId i = 0; i < unit.size(); ++i) wl[i] = work_w[unit.global_ids[i]];
      Eigen::VectorXd rl;
      std::int64_t it = 0;
      switch (unit.kind) {
        case UnitKind::SingletonGroup: rl = solve_singletons(g, unit, wl, params); break;
        case UnitKind::Cac: rl = solve_cac(g, unit, wl, params); break;
        case UnitKind::SccSmall: rl = solve_small_scc(g, unit, wl, params); break;
        case UnitKind::SccLarge: rl = solve_large_scc(g, unit, wl, large_params, it); break;
      }
      for (VertexId i = 0; i < unit.size(); ++i) ranks[unit.global_ids[i]] = rl[i];
      const int64_t e = static_cast<int64_t>(unit.edges.size());
      work += unit.kind == UnitKind::SccLarge ? it * e : e;
      iters += it;
    };
    for (const ScheduleLevel& level : prep.s.levels) {
      if (threads <= 1 || level.units.size() <= 1) {
        for (const auto& u : level.units) solve_one(u);
      } else {
        std::atomic<std::size_t> next{0};
        std::mutex lock;
        std::exception_ptr err;
        auto worker = [&] {
          for (;;) {
            const std::size_t i = next.fetch_add(1);
            if (i >= level.units.size()) return;
            try {
              solve_one(level.units[i]);
            } catch (...) {
              std::lock_guard<std::mutex> hold(lock);
              if (!err) err = std::current_exception();
              return;
            }
          }
        };
        std::vector<std::thread> pool;
        const std::size_t spawn = std::min<std::size_t>(static_cast<std::size_t>(threads), level.units.size());
        for (std::size_t t = 0; t < spawn; ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
        if (err) std::rethrow_exception(err);
      }
      propagate_weights(level.cross_edges, ranks, c, work_w);
      work += static_cast<int64_t>(level.cross_edges.size());
    }
    *ms_out = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (int64_t i = 0; i < wn; ++i) ranks_out[i] = ranks(i);
    *edge_work_out = work.load();
    *large_iters_out = iters.load();
    return 0;
  } catch (...) {
    return fail_from_current();
  }
}


// ---- output formats.  SolveReport::write_text / write_json are the
// reference's own (proj/src/report.cpp, compiled when nlohmann/json is
// available); the CLI's ranks TSV and bench CSV row live in cli.cpp, which
// cannot build here (CLI11 absent), so they are restated from
// proj/src/cli.cpp:80-83 and :271-275.
typedef struct {
  int32_t kind, level, size, reserved;
  int64_t edges, iterations;
  double wall_ms;
} lrref_unit;

static char* dup_string(const std::string& t, int64_t* len) {
  char* b = static_cast<char*>(std::malloc(t.size() + 1));
  std::memcpy(b, t.data(), t.size());
  b[t.size()] = 0;
  *len = static_cast<int64_t>(t.size());
  return b;
}

// fields: the lrref_report scalars; strings method/mode; fmt 0 text, 1 json, 2 bench row
char* lrref_report_format(const lrref_report* r, const char* method, const char* mode, double c, double tol,
                          int keep_loops, int32_t small_threshold, int threads, const lrref_unit* units,
                          int64_t n_units, int fmt, int64_t* len) {
  SolveReport rep;
  rep.method = method;
  rep.mode = mode;
  rep.c = c;
  rep.tol = tol;
  rep.keep_loops = keep_loops != 0;
  rep.small_threshold = small_threshold;
  rep.threads = threads;
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
  for (int64_t i = 0; i < n_units; ++i)
    rep.units.push_back(UnitRecord{static_cast<UnitKind>(units[i].kind), units[i].level, units[i].size,
                                   units[i].edges, units[i].iterations, units[i].wall_ms});
  std::ostringstream out;
  if (fmt == 2) {
    out << std::setprecision(15);
    out << rep.method << (rep.mode == "parallel" ? "_parallel" : "") << ',' << rep.c << ',' << rep.tol << ','
        << rep.total_iterations << ',' << rep.iterative_edge_work << ',' << rep.wall_ms << '\n';
  } else {
#ifdef LRREF_HAVE_REPORT
    if (fmt == 0) rep.write_text(out);
    else rep.write_json(out);
#else
    return nullptr;
#endif
  }
  return dup_string(out.str(), len);
}

char* lrref_ranks_format(const double* ranks, int64_t n, int64_t* len) {
  std::ostringstream out;
  out << std::setprecision(12);
  for (int64_t v = 0; v < n; ++v) out << v << '\t' << ranks[v] << '\n';
  return dup_string(out.str(), len);
}

void lrref_string_free(char* p) { std::free(p); }


// The reference's unit solvers (proj/src/solvers.cpp:23-162) on a unit given
// as global ids + local edges: kind 0 singletons, 1 cac, 2 small, 3 large.
int lrref_solve_unit(void* gp, int kind, const int32_t* ids, int32_t m, const int32_t* es, const int32_t* ed,
                     int64_t ne, const double* w, double c, double tol, double* out, int64_t* iters,
                     int64_t* visits) {
  try {
    const Graph& g = *static_cast<Graph*>(gp);
    SolveUnit unit;
    unit.kind = static_cast<UnitKind>(kind);
    unit.global_ids.assign(ids, ids + m);
    for (int64_t i = 0; i < ne; ++i) unit.edges.emplace_back(es[i], ed[i]);
    const Eigen::VectorXd wl = to_vec(w, m);
    const SolverParams params{c, tol};
    Eigen::VectorXd r;
    std::int64_t it = 0;
    EdgeId vis = 0;
    switch (kind) {
      case 0: r = solve_singletons(g, unit, wl, params); break;
      case 1: r = solve_cac(g, unit, wl, params, &vis); break;
      case 2: r = solve_small_scc(g, unit, wl, params); break;
      default: r = solve_large_scc(g, unit, wl, params, it); break;
    }
    for (int32_t i = 0; i < m; ++i) out[i] = r(i);
    *iters = it;
    *visits = vis;
    return 0;
  } catch (...) {
    return fail_from_current();
  }
}


// solve_large_scc with PowerSeriesStats (solvers.cpp:128-162).
int lrref_large_scc_stats(void* gp, const int32_t* ids, int32_t m, const int32_t* es, const int32_t* ed, int64_t ne,
                          const double* w, double c, double tol, double* out, int64_t* iters, double* l1,
                          int64_t l1cap, int64_t* l1len, double* mn) {
  try {
    const Graph& g = *static_cast<Graph*>(gp);
    SolveUnit unit;
    unit.kind = UnitKind::SccLarge;
    unit.global_ids.assign(ids, ids + m);
    for (int64_t i = 0; i < ne; ++i) unit.edges.emplace_back(es[i], ed[i]);
    PowerSeriesStats st;
    std::int64_t it = 0;
    const Eigen::VectorXd r = solve_large_scc(g, unit, to_vec(w, m), SolverParams{c, tol}, it, &st);
    for (int32_t i = 0; i < m; ++i) out[i] = r(i);
    *iters = it;
    const int64_t k = std::min<int64_t>(l1cap, static_cast<int64_t>(st.increment_l1_norms.size()));
    for (int64_t i = 0; i < k; ++i) l1[i] = st.increment_l1_norms[static_cast<std::size_t>(i)];
    *l1len = static_cast<int64_t>(st.increment_l1_norms.size());
    *mn = st.min_increment_entry;
    return 0;
  } catch (...) {
    return fail_from_current();
  }
}

}  // extern "C"
