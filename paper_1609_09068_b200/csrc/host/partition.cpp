// SCC/CAC partition: iterative Tarjan with level tracking and the one-pass
// CAC absorption rule (paper Theorem 1; reference proj/src/partition.cpp:52-145),
// union-find with union by depth + path compression
// (proj/include/levelrank/union_find.hpp:11-45), dense ids by first appearance
// and a min-level shift (partition.cpp:23-50).  Written as one flat loop over
// an explicit (vertex, edge cursor) stack with all per-vertex state in
// contiguous int32/uint8 arrays; the work counters follow the reference's
// definitions so PartitionStats match exactly.
#include "levelrank/partition.hpp"

#include <algorithm>
#include <cstdint>
#include <vector>

namespace levelrank {
inline namespace b200 {
namespace {

struct DisjointSets {
  std::vector<std::int32_t> parent;
  std::vector<std::uint8_t> depth;
  explicit DisjointSets(std::int32_t n) : parent(static_cast<std::size_t>(n)), depth(static_cast<std::size_t>(n), 1) {
    for (std::int32_t i = 0; i < n; ++i) parent[static_cast<std::size_t>(i)] = i;
  }
  std::int32_t find(std::int32_t x) {
    std::int32_t r = x;
    while (parent[static_cast<std::size_t>(r)] != r) r = parent[static_cast<std::size_t>(r)];
    while (parent[static_cast<std::size_t>(x)] != r) {
      const std::int32_t nx = parent[static_cast<std::size_t>(x)];
      parent[static_cast<std::size_t>(x)] = r;
      x = nx;
    }
    return r;
  }
  void unite(std::int32_t a, std::int32_t b) {
    a = find(a);
    b = find(b);
    if (a == b) return;
    if (depth[static_cast<std::size_t>(a)] < depth[static_cast<std::size_t>(b)]) std::swap(a, b);
    parent[static_cast<std::size_t>(b)] = a;
    if (depth[static_cast<std::size_t>(a)] == depth[static_cast<std::size_t>(b)]) ++depth[static_cast<std::size_t>(a)];
  }
};

constexpr std::uint8_t kDone = 1;  // component finished ("assigned")
constexpr std::uint8_t kBig = 2;   // member of a size >= 2 SCC

// Per-vertex DFS state in one 16-byte record: a visit costs one cache line
// (the traversal is bound by these random accesses), and the records of the
// next out-neighbours are prefetched while the current edge is handled.
struct VRec {
  std::int32_t order;
  std::int32_t low;
  std::int32_t level;
  std::uint8_t state;
  std::uint8_t pad[3];
};
constexpr EdgeId kPrefetch = 8;

Partition tarjan_partition(const Graph& g, bool absorb_cacs, PartitionStats* stats) {
  const VertexId n = g.vertex_count();
  const EdgeId* off = g.offsets_data();
  const VertexId* tgt = g.targets_data();
  const std::size_t nn = static_cast<std::size_t>(n);
  std::vector<VRec> rec(nn, VRec{-1, 0, 0, 0, {0, 0, 0}});
  DisjointSets sets(n);
  std::vector<VertexId> pending;
  std::vector<std::pair<VertexId, EdgeId>> stack;  // (vertex, next edge index)
  std::vector<VertexId> absorbed;
  pending.reserve(1024);
  stack.reserve(1024);
  PartitionStats st;
  std::int32_t clock = 0;
  auto R = [&](VertexId v) -> VRec& { return rec[static_cast<std::size_t>(v)]; };

  // the level/low update of the reference's update_from (partition.cpp:67-74)
  auto relax = [&](VertexId v, VertexId w) {
    VRec& a = R(v);
    const VRec& b = R(w);
    if (b.state & kDone) {
      a.level = std::max(a.level, b.level + 1);
    } else {
      a.level = std::max(a.level, b.level);
      a.low = std::min(a.low, b.low);
    }
  };
  auto open = [&](VertexId v) {
    VRec& a = R(v);
    a.order = a.low = clock++;
    a.level = 1;
    pending.push_back(v);
    stack.emplace_back(v, off[v]);
    for (EdgeId e = off[v]; e < off[v + 1] && e < off[v] + kPrefetch; ++e) __builtin_prefetch(&rec[static_cast<std::size_t>(tgt[e])]);
  };
  // component root bookkeeping (partition.cpp:76-113)
  auto close = [&](VertexId v) {
    ++st.finish_calls;
    VRec& rv = R(v);
    if (rv.low != rv.order) return;
    std::size_t first = pending.size();
    while (pending[--first] != v) {
    }
    const std::size_t members = pending.size() - first;
    const std::int32_t lv = rv.level;
    for (std::size_t i = first; i < pending.size(); ++i) {
      const VertexId m = pending[i];
      R(m).state = kDone | kBig;
      R(m).level = lv;
      sets.unite(v, m);
    }
    pending.resize(first);
    if (members != 1) return;
    rv.state = kDone;
    if (!absorb_cacs) return;
    absorbed.clear();
    const std::int32_t below = rv.level - 1;
    for (EdgeId e = off[v]; e < off[v + 1]; ++e) {
      ++st.merge_scan_edge_visits;
      const VertexId w = tgt[e];
      if (e + kPrefetch < off[v + 1]) __builtin_prefetch(&rec[static_cast<std::size_t>(tgt[e + kPrefetch])]);
      if (w == v || R(w).level != below) continue;
      if (R(w).state & kBig) return;  // an SCC on the next level vetoes
      absorbed.push_back(w);
    }
    if (absorbed.empty()) return;
    rv.level = below;
    for (const VertexId w : absorbed) sets.unite(v, w);
  };

  for (VertexId s = 0; s < n; ++s) {
    if (R(s).order >= 0) continue;
    open(s);
    while (!stack.empty()) {
      auto& top = stack.back();
      const VertexId v = top.first;
      const EdgeId end = off[v + 1];
      if (top.second < end) {
        const EdgeId e = top.second++;
        const VertexId w = tgt[e];
        if (e + kPrefetch < end) __builtin_prefetch(&rec[static_cast<std::size_t>(tgt[e + kPrefetch])]);
        ++st.explore_edge_visits;
        if (w == v) continue;
        if (R(w).order < 0)
          open(w);
        else
          relax(v, w);
        continue;
      }
      stack.pop_back();
      close(v);
      if (!stack.empty()) relax(stack.back().first, v);
    }
  }
  if (stats) *stats = st;

  Partition p;
  p.comp_of.assign(nn, -1);
  std::vector<VertexId> id_of_root(nn, -1);
  for (VertexId v = 0; v < n; ++v) {
    const VertexId r = sets.find(v);
    VertexId& id = id_of_root[static_cast<std::size_t>(r)];
    if (id < 0) {
      id = static_cast<VertexId>(p.kinds.size());
      p.kinds.push_back((rec[static_cast<std::size_t>(r)].state & kBig) ? ComponentKind::Scc : ComponentKind::Cac);
      p.levels.push_back(rec[static_cast<std::size_t>(r)].level);
      p.sizes.push_back(0);
    }
    p.comp_of[static_cast<std::size_t>(v)] = id;
    ++p.sizes[static_cast<std::size_t>(id)];
  }
  if (!p.levels.empty()) {
    const std::int32_t lo = *std::min_element(p.levels.begin(), p.levels.end());
    for (auto& l : p.levels) l -= lo;
    p.max_level = *std::max_element(p.levels.begin(), p.levels.end());
  }
  return p;
}

}  // namespace

Partition find_components(const Graph& g, PartitionStats* stats) { return tarjan_partition(g, true, stats); }

Partition find_components_scc_only(const Graph& g) { return tarjan_partition(g, false, nullptr); }

std::vector<CanonicalComponent> canonical_components(const Partition& p) {
  std::vector<CanonicalComponent> cs(p.component_count());
  for (std::size_t c = 0; c < cs.size(); ++c) {
    cs[c].kind = p.kinds[c];
    cs[c].level = p.levels[c];
  }
  for (std::size_t v = 0; v < p.comp_of.size(); ++v)
    cs[static_cast<std::size_t>(p.comp_of[v])].members.push_back(static_cast<VertexId>(v));
  std::sort(cs.begin(), cs.end());
  return cs;
}

std::vector<std::uint8_t> big_scc_flags(const Partition& p) {
  std::vector<std::uint8_t> f(p.comp_of.size(), 0);
  for (std::size_t v = 0; v < f.size(); ++v)
    f[v] = p.kinds[static_cast<std::size_t>(p.comp_of[v])] == ComponentKind::Scc;
  return f;
}

PartitionCensus census(const Partition& p) {
  PartitionCensus c;
  c.components = static_cast<std::int64_t>(p.component_count());
  c.max_level = p.max_level;
  c.level_count = p.max_level + 1;
  c.components_per_level.assign(static_cast<std::size_t>(p.max_level + 1), 0);
  VertexId largest = 0;
  for (std::size_t i = 0; i < p.component_count(); ++i) {
    if (p.kinds[i] == ComponentKind::Scc) {
      ++c.scc_components;
    } else {
      ++c.cac_components;
      if (p.sizes[i] == 1) ++c.singleton_cacs;
    }
    ++c.components_per_level[static_cast<std::size_t>(p.levels[i])];
    if (p.sizes[i] > largest) {
      largest = p.sizes[i];
      c.largest_kind = p.kinds[i];
    }
  }
  c.largest_component = largest;
  // size histogram over (bound/2, bound], bounds 1, 2, 4, ...
  std::vector<std::int64_t> bins;
  for (const VertexId s : p.sizes) {
    std::size_t b = 0;
    while ((VertexId{1} << b) < s) ++b;
    if (bins.size() <= b) bins.resize(b + 1, 0);
    ++bins[b];
  }
  for (std::size_t b = 0; b < bins.size(); ++b) c.size_histogram.emplace_back(VertexId{1} << b, bins[b]);
  return c;
}

}  // namespace b200
}  // namespace levelrank
