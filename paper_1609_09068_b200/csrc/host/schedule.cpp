// Level-major schedule (reference-shaped, proj/src/schedule.cpp:32-137) and the
// device Layout the GPU path consumes.
#include "levelrank/schedule.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <numeric>
#include <stdexcept>
#include <thread>

#include "parallel.hpp"
#include "plan_internal.hpp"

namespace levelrank {
inline namespace b200 {
namespace {


// Components in schedule order: level desc, size desc, id asc (two stable
// parallel radix passes: by size, then by level).
std::vector<VertexId> ordered_components(const Partition& p, VertexId) {
  const VertexId k = static_cast<VertexId>(p.component_count());
  std::vector<VertexId> comps(static_cast<std::size_t>(k));
  std::iota(comps.begin(), comps.end(), 0);
  detail::stable_radix_sort(comps.data(), k, [&](VertexId c) {
    return ~static_cast<std::uint32_t>(p.sizes[static_cast<std::size_t>(c)]);
  });
  detail::stable_radix_sort(comps.data(), k, [&](VertexId c) {
    return ~static_cast<std::uint32_t>(p.levels[static_cast<std::size_t>(c)]);
  });
  return comps;
}

// Members of every component, ascending vertex id (CSR by component).  The
// offsets are the scan of the sizes; a single-vertex component's member goes
// straight to its slot, and only the vertices of larger components (in vertex
// order) are sorted by component, stably -- the slots of those components, in
// slot order, take the sorted vertices one to one.
void component_members(const Partition& p, std::vector<std::int64_t>& begin, std::vector<VertexId>& mem) {
  const std::size_t k = p.component_count(), n = p.comp_of.size();
  begin.resize(k + 1);
  begin[k] = 0;
  uvector<std::int64_t> singles_before(k + 1);  // single-vertex components with a smaller id
  singles_before[k] = 0;
  detail::parallel_chunks(static_cast<std::int64_t>(k), [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t c = b; c < e; ++c) {
      begin[static_cast<std::size_t>(c)] = p.sizes[static_cast<std::size_t>(c)];
      singles_before[static_cast<std::size_t>(c)] = p.sizes[static_cast<std::size_t>(c)] == 1;
    }
  });
  detail::exclusive_scan_inplace(begin.data(), static_cast<std::int64_t>(k) + 1);
  detail::exclusive_scan_inplace(singles_before.data(), static_cast<std::int64_t>(k) + 1);
  mem.resize(n);
  const int T = host_threads();
  std::vector<uvector<VertexId>> found(static_cast<std::size_t>(T));
  detail::parallel_chunks(static_cast<std::int64_t>(n), [&](int th, std::int64_t b, std::int64_t e) {
    auto& mine = found[static_cast<std::size_t>(th)];
    for (std::int64_t v = b; v < e; ++v) {
      const std::size_t c = static_cast<std::size_t>(p.comp_of[static_cast<std::size_t>(v)]);
      if (p.sizes[c] == 1) mem[static_cast<std::size_t>(begin[c])] = static_cast<VertexId>(v);
      else mine.push_back(static_cast<VertexId>(v));
    }
  });
  std::vector<std::size_t> at(static_cast<std::size_t>(T) + 1, 0);
  for (int t = 0; t < T; ++t) at[static_cast<std::size_t>(t) + 1] = at[static_cast<std::size_t>(t)] + found[static_cast<std::size_t>(t)].size();
  uvector<VertexId> multi(at[static_cast<std::size_t>(T)]);  // chunks are ascending vertex ranges: vertex order
  detail::parallel_chunks(T, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t t = b; t < e; ++t)
      std::copy(found[static_cast<std::size_t>(t)].begin(), found[static_cast<std::size_t>(t)].end(), multi.begin() + static_cast<std::ptrdiff_t>(at[static_cast<std::size_t>(t)]));
  }, 1);
  detail::stable_radix_sort(multi.data(), static_cast<std::int64_t>(multi.size()), [&](VertexId v) {
    return static_cast<std::uint32_t>(p.comp_of[static_cast<std::size_t>(v)]);
  });
  detail::parallel_chunks(static_cast<std::int64_t>(multi.size()), [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t i = b; i < e; ++i) {
      // slot = position among the slots of multi-vertex components + the single-vertex slots before it
      const VertexId v = multi[static_cast<std::size_t>(i)];
      mem[static_cast<std::size_t>(i + singles_before[static_cast<std::size_t>(p.comp_of[static_cast<std::size_t>(v)])])] = v;
    }
  });
}

// One unit of the plan: a multi-vertex component, or a level's singletons.
struct UnitPlan {
  UnitKind kind;
  std::int32_t level;
  VertexId comp;  // -1: singleton group
  VertexId size;
};

// Units per level in schedule order, singleton group slotted so sizes stay
// non-increasing (schedule.cpp:58-110).  Fills per-level begin offsets.
std::vector<UnitPlan> plan_units(const Partition& p, const std::vector<VertexId>& comps, VertexId threshold,
                                 std::vector<std::int32_t>& level_unit_begin,
                                 std::vector<std::vector<VertexId>>& singles_of_level,
                                 const std::vector<std::int64_t>& mbegin, const std::vector<VertexId>& mem) {
  const std::int32_t nl = p.max_level + 1;
  level_unit_begin.assign(static_cast<std::size_t>(nl) + 1, 0);
  singles_of_level.assign(static_cast<std::size_t>(nl), {});
  std::vector<UnitPlan> units;
  std::size_t walk = 0;
  while (walk < comps.size()) {
    const std::int32_t level = p.levels[static_cast<std::size_t>(comps[walk])];
    const std::size_t li = static_cast<std::size_t>(p.max_level - level);
    level_unit_begin[li] = static_cast<std::int32_t>(units.size());
    const std::size_t first = units.size();
    auto& singles = singles_of_level[li];
    while (walk < comps.size() && p.levels[static_cast<std::size_t>(comps[walk])] == level) {
      const VertexId c = comps[walk++];
      const VertexId sz = p.sizes[static_cast<std::size_t>(c)];
      if (sz == 1) {
        singles.push_back(mem[static_cast<std::size_t>(mbegin[static_cast<std::size_t>(c)])]);
        continue;
      }
      const UnitKind kind = p.kinds[static_cast<std::size_t>(c)] == ComponentKind::Cac ? UnitKind::Cac
                            : sz < threshold                                          ? UnitKind::SccSmall
                                                                                      : UnitKind::SccLarge;
      units.push_back({kind, level, c, sz});
    }
    if (!singles.empty()) {
      // comps of equal level and size come in id order, and ids follow each
      // component's smallest vertex: the singletons are usually sorted already
      if (!std::is_sorted(singles.begin(), singles.end())) std::sort(singles.begin(), singles.end());
      const VertexId gs = static_cast<VertexId>(singles.size());
      auto at = std::find_if(units.begin() + static_cast<std::ptrdiff_t>(first), units.end(),
                             [&](const UnitPlan& u) { return u.size < gs; });
      units.insert(at, UnitPlan{UnitKind::SingletonGroup, level, -1, gs});
    }
  }
  level_unit_begin[static_cast<std::size_t>(nl)] = static_cast<std::int32_t>(units.size());
  for (std::int32_t i = nl - 1; i >= 0; --i)
    level_unit_begin[static_cast<std::size_t>(i)] =
        std::min(level_unit_begin[static_cast<std::size_t>(i)], level_unit_begin[static_cast<std::size_t>(i) + 1]);
  return units;
}

}  // namespace

std::vector<VertexId> schedule_permutation(const Partition& p) {
  const VertexId n = static_cast<VertexId>(p.comp_of.size());
  std::vector<VertexId> perm(static_cast<std::size_t>(n), 0);
  if (n == 0) return perm;
  const auto comps = ordered_components(p, n);
  std::vector<std::int64_t> mb;
  std::vector<VertexId> mem;
  component_members(p, mb, mem);
  VertexId pos = 0;
  for (const VertexId c : comps)
    for (std::int64_t j = mb[static_cast<std::size_t>(c)]; j < mb[static_cast<std::size_t>(c) + 1]; ++j)
      perm[static_cast<std::size_t>(mem[static_cast<std::size_t>(j)])] = pos++;
  return perm;
}

Schedule build_schedule(const Graph& g, const Partition& p, VertexId small_threshold) {
  if (small_threshold < 1) throw std::invalid_argument("small_threshold must be at least 1");
  const VertexId n = g.vertex_count();
  Schedule s;
  if (n == 0) return s;
  const auto comps = ordered_components(p, n);
  std::vector<std::int64_t> mb;
  std::vector<VertexId> mem;
  component_members(p, mb, mem);
  s.permutation = schedule_permutation(p);
  std::vector<std::int32_t> lub;
  std::vector<std::vector<VertexId>> singles;
  const auto plan = plan_units(p, comps, small_threshold, lub, singles, mb, mem);
  const std::size_t nl = static_cast<std::size_t>(p.max_level) + 1;
  s.levels.resize(nl);
  std::vector<VertexId> local_of(static_cast<std::size_t>(n));
  std::vector<SolveUnit*> flat;  // every unit, schedule order
  for (std::size_t li = 0; li < nl; ++li) {
    auto& L = s.levels[li];
    L.level = p.max_level - static_cast<std::int32_t>(li);
    L.units.resize(static_cast<std::size_t>(lub[li + 1] - lub[li]));
    for (std::int32_t ui = lub[li]; ui < lub[li + 1]; ++ui) {
      const UnitPlan& up = plan[static_cast<std::size_t>(ui)];
      SolveUnit& u = L.units[static_cast<std::size_t>(ui - lub[li])];
      u.kind = up.kind;
      u.level = up.level;
      if (up.comp >= 0)
        u.global_ids.assign(mem.begin() + mb[static_cast<std::size_t>(up.comp)],
                            mem.begin() + mb[static_cast<std::size_t>(up.comp) + 1]);
      else
        u.global_ids = singles[li];
      flat.push_back(&u);
    }
  }
  // Intra edges unit by unit (in parallel): the unit's vertices ascending and
  // each row's targets ascending give the (local src, local dst) order the
  // reference's single pass over all vertices produces (schedule.cpp:112-135).
  const bool keep = g.loop_policy() == LoopPolicy::Keep;
  std::atomic<EdgeId> intra{0}, dropped{0};
  detail::parallel_dynamic(static_cast<std::int64_t>(flat.size()), 64, [&](std::int64_t b, std::int64_t e) {
    EdgeId li = 0, ld = 0;
    for (std::int64_t k = b; k < e; ++k) {
      SolveUnit& u = *flat[static_cast<std::size_t>(k)];
      for (std::size_t a = 0; a < u.global_ids.size(); ++a) local_of[static_cast<std::size_t>(u.global_ids[a])] = static_cast<VertexId>(a);
      for (std::size_t a = 0; a < u.global_ids.size(); ++a) {
        const VertexId v = u.global_ids[a];
        const VertexId cv = p.comp_of[static_cast<std::size_t>(v)];
        for (const VertexId t : g.out_neighbors(v)) {
          if (t == v) {
            if (keep) u.edges.emplace_back(static_cast<VertexId>(a), static_cast<VertexId>(a));
            else ++ld;
          } else if (p.comp_of[static_cast<std::size_t>(t)] == cv) {
            u.edges.emplace_back(static_cast<VertexId>(a), local_of[static_cast<std::size_t>(t)]);
          }
        }
      }
      li += static_cast<EdgeId>(u.edges.size());
    }
    intra += li;
    dropped += ld;
  });
  // Cross edges per source level (in parallel over levels), sources ascending.
  std::atomic<EdgeId> cross{0};
  detail::parallel_dynamic(static_cast<std::int64_t>(nl), 1, [&](std::int64_t b, std::int64_t e) {
    for (std::int64_t li = b; li < e; ++li) {
      auto& L = s.levels[static_cast<std::size_t>(li)];
      std::vector<VertexId> sources;
      for (const SolveUnit& u : L.units) sources.insert(sources.end(), u.global_ids.begin(), u.global_ids.end());
      std::sort(sources.begin(), sources.end());
      for (const VertexId v : sources) {
        const VertexId cv = p.comp_of[static_cast<std::size_t>(v)];
        for (const VertexId t : g.out_neighbors(v))
          if (t != v && p.comp_of[static_cast<std::size_t>(t)] != cv) L.cross_edges.push_back({v, t, g.walk_out_degree(v)});
      }
      cross += static_cast<EdgeId>(L.cross_edges.size());
    }
  });
  s.intra_edge_count = intra;
  s.dropped_loop_count = dropped;
  s.cross_edge_count = cross;
  return s;
}

namespace {
constexpr std::int64_t kParallelSortRows = 1 << 16;  // SccLarge units above this sort their rows in parallel
Layout build_layout_impl(const Graph& g, const Partition& p, VertexId small_threshold, const detail::InEdges* in);
}

Layout build_layout(const Graph& g, const Partition& p, VertexId small_threshold) {
  return build_layout_impl(g, p, small_threshold, nullptr);
}

namespace detail {
Layout build_layout_from(const Graph& g, const Partition& p, VertexId small_threshold, const InEdges& in) {
  return build_layout_impl(g, p, small_threshold, &in);
}
}  // namespace detail

namespace {
// in: the graph's in-edge lists when the partition already built them (then
// the pull lists are gathered per row instead of transposing every edge again)
Layout build_layout_impl(const Graph& g, const Partition& p, VertexId small_threshold, const detail::InEdges* in) {
  if (small_threshold < 1) throw std::invalid_argument("small_threshold must be at least 1");
  const VertexId n = g.vertex_count();
  const std::size_t nn = static_cast<std::size_t>(n);
  const bool keep = g.loop_policy() == LoopPolicy::Keep;
  Layout L;
  L.n = n;
  L.max_level = p.max_level;
  L.keep_loops = keep;
  L.level_row_begin.assign(1, 0);
  L.level_unit_begin.assign(1, 0);
  L.unit_row_begin.assign(1, 0);
  L.xptr.assign(1, 0);
  L.iptr.assign(1, 0);
  if (n == 0) return L;
  const EdgeId* off = g.offsets_data();
  const VertexId* tgt = g.targets_data();
  const std::uint8_t* lp = g.loop_data();
  const auto& comp_of = p.comp_of;

  detail::PhaseClock clk;
  // component order and member lists depend only on the partition: side by side
  // (the second one's parallel loops find the pool busy and spawn their threads)
  std::vector<VertexId> comps;
  std::exception_ptr side_error;
  std::thread side([&] {
    try {
      comps = ordered_components(p, n);
    } catch (...) {
      side_error = std::current_exception();
    }
  });
  std::vector<std::int64_t> mb;
  std::vector<VertexId> mem;
  try {
    component_members(p, mb, mem);
  } catch (...) {
    side.join();
    throw;
  }
  side.join();
  if (side_error) std::rethrow_exception(side_error);

  std::vector<std::vector<VertexId>> singles;
  const auto plan = plan_units(p, comps, small_threshold, L.level_unit_begin, singles, mb, mem);
  const std::size_t nu = plan.size();
  clk.mark("components + unit plan");
  const std::int32_t nl = p.max_level + 1;

  // unit of every vertex, local index (= position in ascending members)
  uvector<std::int32_t> unit_of(nn), local_of(nn);  // every vertex is in a unit: written below
  std::vector<std::int64_t> unit_mem_begin(nu + 1, 0);  // into `umem`
  uvector<VertexId> umem(nn);
  {
    // offsets first (one step per unit), then the members of every unit copied and
    // numbered in parallel: small units several per task, the giant SCC and the
    // levels' singleton groups (millions of members each) split over the threads
    std::vector<const VertexId*> unit_src(nu);
    std::int64_t pos = 0;
    for (std::int32_t li = 0; li < nl; ++li)
      for (std::int32_t ui = L.level_unit_begin[static_cast<std::size_t>(li)];
           ui < L.level_unit_begin[static_cast<std::size_t>(li) + 1]; ++ui) {
        const UnitPlan& up = plan[static_cast<std::size_t>(ui)];
        unit_mem_begin[static_cast<std::size_t>(ui)] = pos;
        if (up.comp >= 0) {
          unit_src[static_cast<std::size_t>(ui)] = mem.data() + mb[static_cast<std::size_t>(up.comp)];
          pos += mb[static_cast<std::size_t>(up.comp) + 1] - mb[static_cast<std::size_t>(up.comp)];
        } else {
          unit_src[static_cast<std::size_t>(ui)] = singles[static_cast<std::size_t>(li)].data();
          pos += static_cast<std::int64_t>(singles[static_cast<std::size_t>(li)].size());
        }
      }
    unit_mem_begin[nu] = pos;
    constexpr std::int64_t kBigUnit = 1 << 18;
    auto fill = [&](std::int64_t u, std::int64_t j0, std::int64_t j1) {
      const std::int64_t base = unit_mem_begin[static_cast<std::size_t>(u)];
      const VertexId* src = unit_src[static_cast<std::size_t>(u)];
      for (std::int64_t j = j0; j < j1; ++j) {
        const VertexId v = src[j];
        umem[static_cast<std::size_t>(base + j)] = v;
        unit_of[static_cast<std::size_t>(v)] = static_cast<std::int32_t>(u);
        local_of[static_cast<std::size_t>(v)] = static_cast<std::int32_t>(j);
      }
    };
    detail::parallel_dynamic(static_cast<std::int64_t>(nu), 256, [&](std::int64_t b, std::int64_t e) {
      for (std::int64_t u = b; u < e; ++u) {
        const std::int64_t m = unit_mem_begin[static_cast<std::size_t>(u) + 1] - unit_mem_begin[static_cast<std::size_t>(u)];
        if (m <= kBigUnit) fill(u, 0, m);
      }
    });
    for (std::size_t u = 0; u < nu; ++u) {
      const std::int64_t m = unit_mem_begin[u + 1] - unit_mem_begin[u];
      if (m > kBigUnit)
        detail::parallel_chunks(m, [&](int, std::int64_t b, std::int64_t e) { fill(static_cast<std::int64_t>(u), b, e); });
    }
  }

  clk.mark("unit_of / local_of");
  // CAC units: Kahn pass of solve_cac (solvers.cpp:43-83) to get each vertex's
  // dequeue position and its depth (longest path from the unit's sources).
  uvector<std::int32_t> kahn_pos(nn), depth(nn);  // written and read for CAC vertices only
  std::vector<std::int32_t> unit_depths(nu, 0);
  std::atomic<bool> cycle{false};
  detail::parallel_dynamic(static_cast<std::int64_t>(nu), 64, [&](std::int64_t b, std::int64_t e) {
    std::vector<std::int32_t> adj_off, adj, indeg, queue, dep;
    for (std::int64_t u = b; u < e; ++u) {
      if (plan[static_cast<std::size_t>(u)].kind != UnitKind::Cac) continue;
      const std::int64_t m0 = unit_mem_begin[static_cast<std::size_t>(u)];
      const std::int32_t m = static_cast<std::int32_t>(unit_mem_begin[static_cast<std::size_t>(u) + 1] - m0);
      const VertexId c = comp_of[static_cast<std::size_t>(umem[static_cast<std::size_t>(m0)])];
      adj_off.assign(static_cast<std::size_t>(m) + 1, 0);
      indeg.assign(static_cast<std::size_t>(m), 0);
      adj.clear();
      for (std::int32_t a = 0; a < m; ++a) {
        const VertexId ga = umem[static_cast<std::size_t>(m0 + a)];
        for (EdgeId k = off[ga]; k < off[ga + 1]; ++k) {
          const VertexId gb = tgt[k];
          if (gb == ga || comp_of[static_cast<std::size_t>(gb)] != c) continue;
          const std::int32_t lb = local_of[static_cast<std::size_t>(gb)];
          adj.push_back(lb);
          ++indeg[static_cast<std::size_t>(lb)];
        }
        adj_off[static_cast<std::size_t>(a) + 1] = static_cast<std::int32_t>(adj.size());
      }
      queue.clear();
      dep.assign(static_cast<std::size_t>(m), 0);
      for (std::int32_t a = 0; a < m; ++a)
        if (indeg[static_cast<std::size_t>(a)] == 0) queue.push_back(a);
      std::size_t head = 0;
      while (head < queue.size()) {
        const std::int32_t a = queue[head++];
        for (std::int32_t k = adj_off[static_cast<std::size_t>(a)]; k < adj_off[static_cast<std::size_t>(a) + 1]; ++k) {
          const std::int32_t bb = adj[static_cast<std::size_t>(k)];
          dep[static_cast<std::size_t>(bb)] = std::max(dep[static_cast<std::size_t>(bb)], dep[static_cast<std::size_t>(a)] + 1);
          if (--indeg[static_cast<std::size_t>(bb)] == 0) queue.push_back(bb);
        }
      }
      if (static_cast<std::int32_t>(queue.size()) != m) {
        cycle = true;
        continue;
      }
      std::int32_t maxd = 0;
      for (std::int32_t i = 0; i < m; ++i) {
        const VertexId gv = umem[static_cast<std::size_t>(m0 + queue[static_cast<std::size_t>(i)])];
        kahn_pos[static_cast<std::size_t>(gv)] = i;
        depth[static_cast<std::size_t>(gv)] = dep[static_cast<std::size_t>(queue[static_cast<std::size_t>(i)])];
        maxd = std::max(maxd, dep[static_cast<std::size_t>(queue[static_cast<std::size_t>(i)])]);
      }
      unit_depths[static_cast<std::size_t>(u)] = maxd + 1;
    }
  });

  if (cycle) throw CycleError("cycle inside an acyclic component");
  clk.mark("CAC Kahn passes");

  // rows: units in order; CAC rows by (depth, vertex)
  L.vertex_of.resize(nn);
  L.row_of.resize(nn);
  L.unit_row_begin.assign(nu + 1, 0);
  L.unit_kind.resize(nu);
  L.unit_level.resize(nu);
  L.cac_depth_begin.assign(nu, -1);
  for (std::size_t u = 0; u < nu; ++u) {
    L.unit_row_begin[u] = static_cast<std::int32_t>(unit_mem_begin[u]);
    L.unit_kind[u] = static_cast<std::uint8_t>(plan[u].kind);
    L.unit_level[u] = plan[u].level;
    if (plan[u].kind == UnitKind::Cac) {
      L.cac_depth_begin[u] = static_cast<std::int64_t>(L.depth_ptr.size());
      L.depth_ptr.resize(L.depth_ptr.size() + static_cast<std::size_t>(unit_depths[u]) + 1, 0);
    }
  }
  L.unit_row_begin[nu] = n;
  // Large SCC units: rows (= gather columns) by descending in-unit out-degree,
  // so the most-gathered s values sit together at the head of the unit.
  // one scan of every out-edge: intra-component out-degree per vertex (kept
  // self-loops count, ignored ones are dropped) -> SccLarge row order and the
  // per-unit reference edge counts (unit.edges.size()); cross / dropped totals
  uvector<std::int32_t> unit_out(nn);
  std::atomic<EdgeId> n_intra{0}, n_cross{0}, n_dropped{0};
  const EdgeId m_all = off[n];
  // with the partition's cross-edge bits only the edges that leave their SCC need
  // their components looked up (a clear bit: same SCC, same component)
  const std::uint64_t* xo_bits = in && !in->cross_out.empty() ? in->cross_out.data() : nullptr;
  const std::uint64_t* xi_bits = in && !in->cross_in.empty() ? in->cross_in.data() : nullptr;
  detail::parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
    EdgeId li = 0, lx = 0, ld = 0;
    for (std::int64_t uu = b; uu < e; ++uu) {
      const VertexId u = static_cast<VertexId>(uu);
      const VertexId cu = comp_of[static_cast<std::size_t>(u)];
      std::int32_t k = 0;
      const EdgeId q1 = off[u + 1];
      if (xo_bits) {
        EdgeId self = 0;
        if (lp[u])
          for (EdgeId q = off[u]; q < q1; ++q) self += tgt[q] == u;
        EdgeId leaving = 0, merged = 0;  // out of the SCC; of those, inside the final component
        detail::for_cross_bits(xo_bits, off[u], q1, [&](EdgeId q) {
          ++leaving;
          merged += comp_of[static_cast<std::size_t>(tgt[q])] == cu;
        });
        k = static_cast<std::int32_t>((q1 - off[u]) - self - leaving + merged + (keep ? self : 0));
        if (!keep) ld += self;
        lx += leaving - merged;
        unit_out[static_cast<std::size_t>(u)] = k;
        li += k;
        continue;
      }
      for (EdgeId q = off[u]; q < q1; ++q) {
        const VertexId v = tgt[q];
        if (q + 16 < m_all) __builtin_prefetch(&comp_of[static_cast<std::size_t>(tgt[q + 16])]);
        if (v == u) {
          if (keep) ++k;
          else ++ld;
        } else if (comp_of[static_cast<std::size_t>(v)] == cu) {
          ++k;
        } else {
          ++lx;
        }
      }
      unit_out[static_cast<std::size_t>(u)] = k;
      li += k;
    }
    n_intra += li;
    n_cross += lx;
    n_dropped += ld;
  });
  detail::parallel_dynamic(static_cast<std::int64_t>(nu), 256, [&](std::int64_t b, std::int64_t e) {
    for (std::int64_t uu = b; uu < e; ++uu) {
      const std::size_t u = static_cast<std::size_t>(uu);
      const std::int64_t m0 = unit_mem_begin[u], m1 = unit_mem_begin[u + 1];
      VertexId* rows = L.vertex_of.data() + m0;
      std::copy(umem.begin() + m0, umem.begin() + m1, rows);
      if (plan[u].kind == UnitKind::SccLarge && m1 - m0 <= kParallelSortRows)
        std::stable_sort(rows, rows + (m1 - m0), [&](VertexId a, VertexId bb) {
          return unit_out[static_cast<std::size_t>(a)] > unit_out[static_cast<std::size_t>(bb)];
        });
      if (plan[u].kind == UnitKind::Cac) {
        std::stable_sort(rows, rows + (m1 - m0), [&](VertexId a, VertexId bb) {
          return depth[static_cast<std::size_t>(a)] < depth[static_cast<std::size_t>(bb)];
        });
        std::int32_t* dp = L.depth_ptr.data() + L.cac_depth_begin[u];
        for (std::int64_t r = m0; r < m1; ++r) ++dp[depth[static_cast<std::size_t>(L.vertex_of[static_cast<std::size_t>(r)])] + 1];
        dp[0] = static_cast<std::int32_t>(m0);
        for (std::int32_t d = 0; d < unit_depths[u]; ++d) dp[d + 1] += dp[d];
      }
      if (plan[u].kind == UnitKind::SccLarge && m1 - m0 > kParallelSortRows) continue;  // below
      for (std::int64_t r = m0; r < m1; ++r) L.row_of[static_cast<std::size_t>(L.vertex_of[static_cast<std::size_t>(r)])] = static_cast<VertexId>(r);
    }
  });
  // the giant units: a parallel stable radix sort by descending out-degree
  for (std::size_t u = 0; u < nu; ++u) {
    const std::int64_t m0 = unit_mem_begin[u], m1 = unit_mem_begin[u + 1];
    if (plan[u].kind != UnitKind::SccLarge || m1 - m0 <= kParallelSortRows) continue;
    VertexId* rows = L.vertex_of.data() + m0;
    detail::stable_radix_sort(rows, m1 - m0, [&](VertexId v) {
      return ~static_cast<std::uint32_t>(unit_out[static_cast<std::size_t>(v)]);
    });
    detail::parallel_chunks(m1 - m0, [&](int, std::int64_t b, std::int64_t e) {
      for (std::int64_t r = b; r < e; ++r) L.row_of[static_cast<std::size_t>(rows[r])] = static_cast<VertexId>(m0 + r);
    });
  }
  clk.mark("unit out-degrees + row order");
  L.level_row_begin.assign(static_cast<std::size_t>(nl) + 1, 0);
  for (std::int32_t li = 0; li <= nl; ++li)
    L.level_row_begin[static_cast<std::size_t>(li)] = L.unit_row_begin[static_cast<std::size_t>(L.level_unit_begin[static_cast<std::size_t>(li)])];

  L.deg.resize(nn);
  L.loop.assign(nn, 0);
  detail::parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t r = b; r < e; ++r) {
      const VertexId v = L.vertex_of[static_cast<std::size_t>(r)];
      L.deg[static_cast<std::size_t>(r)] = g.walk_out_degree(v);
      const UnitKind k = plan[static_cast<std::size_t>(unit_of[static_cast<std::size_t>(v)])].kind;
      L.loop[static_cast<std::size_t>(r)] = keep && lp[v] && (k == UnitKind::SingletonGroup || k == UnitKind::Cac);
    }
  });

  // per-unit reference edge counts (unit.edges.size())
  std::vector<EdgeId> uedges(nu, 0);
  detail::parallel_dynamic(static_cast<std::int64_t>(nu), 256, [&](std::int64_t b, std::int64_t e) {
    for (std::int64_t u = b; u < e; ++u) {
      EdgeId s = 0;
      for (std::int64_t j = unit_mem_begin[static_cast<std::size_t>(u)]; j < unit_mem_begin[static_cast<std::size_t>(u) + 1]; ++j)
        s += unit_out[static_cast<std::size_t>(umem[static_cast<std::size_t>(j)])];
      uedges[static_cast<std::size_t>(u)] = s;
    }
  });
  L.intra_edge_count = n_intra;
  L.cross_edge_count = n_cross;
  L.dropped_loop_count = n_dropped;
  L.unit_edges = std::move(uedges);
  clk.mark("deg/loop + edge counts");
  // pull lists (sources as vertex ids, source ascending): intra = CSR 0
  // (kept self-loops only in SCC rows), cross = CSR 1
  uvector<EdgeId> icnt, xcnt;
  if (in) {  // gathered per row from the partition's in-edge lists
    icnt.resize(nn + 1);  // every row written below; [nn] receives the scan total
    xcnt.resize(nn + 1);
    icnt[nn] = xcnt[nn] = 0;
    auto row_loop = [&](VertexId v) {
      const UnitKind k = plan[static_cast<std::size_t>(unit_of[static_cast<std::size_t>(v)])].kind;
      return keep && lp[v] && (k == UnitKind::SccSmall || k == UnitKind::SccLarge);
    };
    // both passes walk vertices in id order, so the in-edge lists stream and
    // the random component lookups are prefetched a fixed distance ahead
    const EdgeId in_end = in->off[nn];
    auto ahead = [&](EdgeId k) {
      if (k + 16 < in_end) __builtin_prefetch(&comp_of[static_cast<std::size_t>(in->src[static_cast<std::size_t>(k + 16)])]);
    };
    detail::parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
      for (std::int64_t vv = b; vv < e; ++vv) {
        const VertexId v = static_cast<VertexId>(vv);
        const VertexId cv = comp_of[static_cast<std::size_t>(v)];
        EdgeId ni = row_loop(v) ? 1 : 0, nx = 0;
        const EdgeId k1 = in->off[static_cast<std::size_t>(v) + 1];
        if (xi_bits) {
          detail::for_cross_bits(xi_bits, in->off[static_cast<std::size_t>(v)], k1, [&](EdgeId k) {
            nx += comp_of[static_cast<std::size_t>(in->src[static_cast<std::size_t>(k)])] != cv;
          });
          ni += (k1 - in->off[static_cast<std::size_t>(v)]) - nx;
        } else {
          for (EdgeId k = in->off[static_cast<std::size_t>(v)]; k < k1; ++k) {
            ahead(k);
            if (comp_of[static_cast<std::size_t>(in->src[static_cast<std::size_t>(k)])] == cv) ++ni;
            else ++nx;
          }
        }
        const std::size_t r = static_cast<std::size_t>(L.row_of[static_cast<std::size_t>(v)]);
        icnt[r] = ni;
        xcnt[r] = nx;
      }
    });
    L.isrc.resize(static_cast<std::size_t>(detail::exclusive_scan_inplace(icnt.data(), static_cast<std::int64_t>(nn) + 1)));
    L.xsrc.resize(static_cast<std::size_t>(detail::exclusive_scan_inplace(xcnt.data(), static_cast<std::int64_t>(nn) + 1)));
    detail::parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
      for (std::int64_t vv = b; vv < e; ++vv) {
        const VertexId v = static_cast<VertexId>(vv);
        const std::size_t r = static_cast<std::size_t>(L.row_of[static_cast<std::size_t>(v)]);
        const VertexId cv = comp_of[static_cast<std::size_t>(v)];
        bool loop_due = row_loop(v);  // a kept self-loop sits at its place in source order
        EdgeId ai = icnt[r], ax = xcnt[r];
        const EdgeId k1 = in->off[static_cast<std::size_t>(v) + 1];
        for (EdgeId k = in->off[static_cast<std::size_t>(v)]; k < k1; ++k) {
          const VertexId src = in->src[static_cast<std::size_t>(k)];
          if (!xi_bits) ahead(k);
          if (loop_due && src > v) {
            L.isrc[static_cast<std::size_t>(ai++)] = v;
            loop_due = false;
          }
          const bool intra = xi_bits && !((xi_bits[k >> 6] >> (k & 63)) & 1)
                                 ? true
                                 : comp_of[static_cast<std::size_t>(src)] == cv;
          if (intra) L.isrc[static_cast<std::size_t>(ai++)] = src;
          else L.xsrc[static_cast<std::size_t>(ax++)] = src;
        }
        if (loop_due) L.isrc[static_cast<std::size_t>(ai++)] = v;
      }
    });
  } else {  // one stable bucketed transpose of every out-edge
    // a target's row and component come from one packed 8-byte record
    std::vector<std::uint64_t> rowcomp(nn);
    detail::parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
      for (std::int64_t v = b; v < e; ++v)
        rowcomp[static_cast<std::size_t>(v)] =
            (static_cast<std::uint64_t>(static_cast<std::uint32_t>(comp_of[static_cast<std::size_t>(v)])) << 32) |
            static_cast<std::uint32_t>(L.row_of[static_cast<std::size_t>(v)]);
    });
    uvector<EdgeId> ptrs[2];
    uvector<VertexId> cols[2];
    detail::bucket_csr<2>(
        n, n,
        [&](std::int64_t uu, auto&& sink) {
          const VertexId u = static_cast<VertexId>(uu);
          const std::uint32_t cu = static_cast<std::uint32_t>(comp_of[static_cast<std::size_t>(u)]);
          const UnitKind k = plan[static_cast<std::size_t>(unit_of[static_cast<std::size_t>(u)])].kind;
          const bool scc = k == UnitKind::SccSmall || k == UnitKind::SccLarge;
          const EdgeId q1 = off[u + 1];
          for (EdgeId q = off[u]; q < q1; ++q) {
            const VertexId v = tgt[q];
            if (q + 8 < q1) __builtin_prefetch(&rowcomp[static_cast<std::size_t>(tgt[q + 8])]);
            const std::uint64_t rc = rowcomp[static_cast<std::size_t>(v)];
            const std::int64_t rv = static_cast<std::uint32_t>(rc);
            if (v == u) {
              if (keep && scc) sink(0, rv, u);
            } else {
              sink(static_cast<std::uint32_t>(rc >> 32) == cu ? 0 : 1, rv, u);
            }
          }
        },
        ptrs, cols);
    icnt = std::move(ptrs[0]);
    xcnt = std::move(ptrs[1]);
    L.isrc = std::move(cols[0]);
    L.xsrc = std::move(cols[1]);
  }
  clk.mark("in-edge transpose");
  // per-row ordering = the reference's accumulation order, then vertex -> row
  uvector<std::int32_t> level_idx_of(nn);
  detail::parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t v = b; v < e; ++v)
      level_idx_of[static_cast<std::size_t>(v)] = p.max_level - p.levels[static_cast<std::size_t>(comp_of[static_cast<std::size_t>(v)])];
  });
  detail::parallel_dynamic(n, 2048, [&](std::int64_t b, std::int64_t e) {
    for (std::int64_t r = b; r < e; ++r) {
      const VertexId v = L.vertex_of[static_cast<std::size_t>(r)];
      const UnitKind k = plan[static_cast<std::size_t>(unit_of[static_cast<std::size_t>(v)])].kind;
      VertexId* a = L.isrc.data() + icnt[static_cast<std::size_t>(r)];
      VertexId* ae = L.isrc.data() + icnt[static_cast<std::size_t>(r) + 1];
      if (k == UnitKind::Cac)  // (SCC rows are source-ascending already)
        std::sort(a, ae, [&](VertexId x, VertexId y) { return kahn_pos[static_cast<std::size_t>(x)] < kahn_pos[static_cast<std::size_t>(y)]; });
      for (VertexId* q = a; q < ae; ++q) *q = L.row_of[static_cast<std::size_t>(*q)];
      VertexId* x = L.xsrc.data() + xcnt[static_cast<std::size_t>(r)];
      VertexId* xe = L.xsrc.data() + xcnt[static_cast<std::size_t>(r) + 1];
      std::sort(x, xe, [&](VertexId s1, VertexId s2) {
        const std::int32_t l1 = level_idx_of[static_cast<std::size_t>(s1)], l2 = level_idx_of[static_cast<std::size_t>(s2)];
        return l1 != l2 ? l1 < l2 : s1 < s2;
      });
      for (VertexId* q = x; q < xe; ++q) *q = L.row_of[static_cast<std::size_t>(*q)];
    }
  });
  clk.mark("per-row sorts");
  L.iptr = std::move(icnt);
  L.xptr = std::move(xcnt);
  return L;
}
}  // namespace

Layout build_baseline_layout(const Graph& g) {
  const VertexId n = g.vertex_count();
  const std::size_t nn = static_cast<std::size_t>(n);
  const bool keep = g.loop_policy() == LoopPolicy::Keep;
  Layout L;
  L.n = n;
  L.keep_loops = keep;
  L.level_row_begin.assign(1, 0);
  L.level_unit_begin.assign(1, 0);
  L.unit_row_begin.assign(1, 0);
  L.xptr.assign(1, 0);
  L.iptr.assign(1, 0);
  if (n == 0) return L;
  const EdgeId* off = g.offsets_data();
  const VertexId* tgt = g.targets_data();
  const std::uint8_t* lp = g.loop_data();
  L.max_level = 0;
  L.level_row_begin = {0, n};
  L.level_unit_begin = {0, 1};
  L.unit_row_begin = {0, n};
  L.unit_kind = {static_cast<std::uint8_t>(UnitKind::SccLarge)};
  L.unit_level = {0};
  L.cac_depth_begin = {-1};
  // walk out-degree and in-degree (ignored self-loops excluded)
  std::vector<VertexId> wd(nn);
  std::vector<std::atomic<std::int64_t>> indeg(nn);
  detail::parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t v = b; v < e; ++v) indeg[static_cast<std::size_t>(v)].store(0, std::memory_order_relaxed);
  });
  detail::parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t uu = b; uu < e; ++uu) {
      const VertexId u = static_cast<VertexId>(uu);
      const bool drop = lp[u] && !keep;
      wd[static_cast<std::size_t>(u)] = static_cast<VertexId>(off[u + 1] - off[u]) - (drop ? 1 : 0);
      for (EdgeId k = off[u]; k < off[u + 1]; ++k)
        if (tgt[k] != u || keep) indeg[static_cast<std::size_t>(tgt[k])].fetch_add(1, std::memory_order_relaxed);
    }
  });
  // rows by descending walk out-degree (the most-gathered pushed values
  // first), vertices without in-edges after all others: their rows never
  // change after the first iteration and form one run of empty SpMV rows
  L.vertex_of.resize(nn);
  for (std::size_t v = 0; v < nn; ++v) L.vertex_of[v] = static_cast<VertexId>(v);
  std::stable_sort(L.vertex_of.begin(), L.vertex_of.end(), [&](VertexId a, VertexId b) {
    const bool ea = indeg[static_cast<std::size_t>(a)].load(std::memory_order_relaxed) == 0;
    const bool eb = indeg[static_cast<std::size_t>(b)].load(std::memory_order_relaxed) == 0;
    if (ea != eb) return eb;
    return wd[static_cast<std::size_t>(a)] > wd[static_cast<std::size_t>(b)];
  });
  L.row_of.resize(nn);
  L.deg.resize(nn);
  L.loop.assign(nn, 0);
  L.xptr.assign(nn + 1, 0);
  L.iptr.assign(nn + 1, 0);
  for (std::size_t r = 0; r < nn; ++r) {
    const VertexId v = L.vertex_of[r];
    L.row_of[static_cast<std::size_t>(v)] = static_cast<VertexId>(r);
    L.deg[r] = wd[static_cast<std::size_t>(v)];
    L.iptr[r + 1] = L.iptr[r] + indeg[static_cast<std::size_t>(v)].load(std::memory_order_relaxed);
  }
  // in-edges per row, source ascending (the reference's push order)
  uvector<EdgeId> ptrs[1];
  uvector<VertexId> cols[1];
  detail::bucket_csr<1>(
      n, n,
      [&](std::int64_t uu, auto&& sink) {
        const VertexId u = static_cast<VertexId>(uu);
        const VertexId ru = L.row_of[static_cast<std::size_t>(u)];
        for (EdgeId k = off[u]; k < off[u + 1]; ++k)
          if (tgt[k] != u || keep) sink(0, L.row_of[static_cast<std::size_t>(tgt[k])], ru);
      },
      ptrs, cols);
  L.isrc = std::move(cols[0]);
  const EdgeId m = L.iptr[nn];
  if (ptrs[0][nn] != m) throw std::logic_error("baseline layout: in-edge count mismatch");
  L.unit_edges = {m};
  L.intra_edge_count = m;
  L.cross_edge_count = 0;
  EdgeId dropped = 0;
  if (!keep)
    for (VertexId v = 0; v < n; ++v) dropped += lp[v] ? 1 : 0;
  L.dropped_loop_count = dropped;
  return L;
}

}  // namespace b200
}  // namespace levelrank
