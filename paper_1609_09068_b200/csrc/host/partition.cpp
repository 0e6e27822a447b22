// SCC/CAC partition with levels (paper §3, Theorem 1), computed in parallel.
//
// The reference finds it in one serial pass (proj/src/partition.cpp:52-145:
// iterative Tarjan, level = longest path to a sink over finished components,
// a fresh single-vertex component absorbing the CACs one level down unless an
// SCC sits there, union-find, ids by first appearance, min-level shift at
// :23-50).  Theorem 1 makes that partition unique, so it can be computed in
// any order that respects the component DAG:
//
//   1. SCCs: iterative trimming of vertices with no live in- or out-edge
//      (trivial SCCs), a forward/backward reachability pass from the
//      highest-degree live vertex (the giant SCC of a scale-free graph), a
//      second trim, and a serial Tarjan over what is left (small SCCs);
//   2. levels and CAC absorption: the component DAG is peeled from its sinks
//      in wavefronts (Kahn on cross-edge counts); a component is decided once
//      all its successors are -- its level is 1 + the highest successor level
//      (1 for sinks), and a single-vertex component applies the absorption
//      rule to its out-edges in row order (that scan also yields the
//      reference's merge_scan_edge_visits);
//   3. absorptions are unioned afterwards, ids numbered by each final
//      component's smallest vertex (= first appearance), levels shifted.
//
// Wavefronts are parallel over components and, for a component with many
// members (the giant SCC), over its members.  PartitionStats follow the
// reference's definitions: every out-edge is explored once
// (explore_edge_visits = m), finish runs once per vertex (finish_calls = n).
#include "levelrank/partition.hpp"

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <thread>
#include <vector>

#include "parallel.hpp"
#include "plan_internal.hpp"

namespace levelrank {
inline namespace b200 {
namespace {

using detail::parallel_chunks;
using detail::parallel_dynamic;

template <typename T>
T atomic_sub(T& x, T v) {
  return std::atomic_ref<T>(x).fetch_sub(v, std::memory_order_acq_rel);
}
inline bool claim(std::uint8_t& flag) {
  std::atomic_ref<std::uint8_t> f(flag);
  return f.load(std::memory_order_relaxed) == 0 && f.exchange(1, std::memory_order_acq_rel) == 0;
}

// Work lists filled by many threads: one vector per thread, concatenated.
struct Frontier {
  std::vector<std::vector<std::int32_t>> parts;
  explicit Frontier(int t) : parts(static_cast<std::size_t>(t)) {}
  std::vector<std::int32_t> take() {
    std::size_t total = 0;
    for (const auto& p : parts) total += p.size();
    std::vector<std::int32_t> out;
    out.reserve(total);
    for (auto& p : parts) {
      out.insert(out.end(), p.begin(), p.end());
      p.clear();
    }
    return out;
  }
};

// One bit per vertex, set/cleared atomically.
struct Bits {
  std::vector<std::uint64_t> w;
  explicit Bits(std::size_t n) : w((n + 63) / 64, 0) {}
  bool get(VertexId v) const { return (w[static_cast<std::size_t>(v) >> 6] >> (v & 63)) & 1u; }
  // true if this call set the bit
  bool set_atomic(VertexId v) {
    const std::uint64_t bit = std::uint64_t{1} << (v & 63);
    std::atomic_ref<std::uint64_t> a(w[static_cast<std::size_t>(v) >> 6]);
    return !(a.load(std::memory_order_relaxed) & bit) && !(a.fetch_or(bit, std::memory_order_relaxed) & bit);
  }
  void clear_atomic(VertexId v) {
    std::atomic_ref<std::uint64_t>(w[static_cast<std::size_t>(v) >> 6])
        .fetch_and(~(std::uint64_t{1} << (v & 63)), std::memory_order_relaxed);
  }
};

// parallel_chunks with the thread index bounded by host_threads(): the items
// are components or vertices whose edge scans are random-access bound, so even
// a deep DAG's small wavefronts (~2k components) are spread over every thread
// (the pool keeps a phase's overhead to microseconds)
template <typename F>
void for_items(const std::vector<std::int32_t>& items, F&& f, std::int64_t grain) {
  parallel_chunks(static_cast<std::int64_t>(items.size()),
                  [&](int th, std::int64_t b, std::int64_t e) {
                    for (std::int64_t i = b; i < e; ++i) f(th, items[static_cast<std::size_t>(i)]);
                  },
                  grain);
}
// items per thread: small on big graphs (each item's scan misses cache), large
// on small graphs (where a phase is shorter than waking the workers)
inline std::int64_t item_grain(std::int64_t n) { return n >= (1 << 22) ? 64 : 4096; }

struct Adjacency {
  const EdgeId* off;
  const VertexId* tgt;
  const std::uint8_t* loop;  // vertex has a self-loop among its out-edges
  uvector<EdgeId> in_off;  // in-edges (self-loops left out), source-ascending rows
  uvector<VertexId> in_src;
};

// ------------------------------------------------------------- 1. SCC labels
class SccFinder {
 public:
  SccFinder(VertexId n, const Adjacency& a, detail::PhaseClock& clk)
      : n_(n), a_(a), clk_(clk), label_(detail::filled<VertexId>(static_cast<std::size_t>(n), -1)) {}

  // label[v] = a representative vertex of v's SCC
  uvector<VertexId> run() {
    const std::size_t nn = static_cast<std::size_t>(n_);
    din_.resize(nn);  // both written for every vertex below
    dout_.resize(nn);
    queued_ = detail::filled<std::uint8_t>(nn, 0);
    parallel_chunks(n_, [&](int, std::int64_t b, std::int64_t e) {
      for (std::int64_t v = b; v < e; ++v) {
        din_[static_cast<std::size_t>(v)] = static_cast<std::int32_t>(a_.in_off[static_cast<std::size_t>(v) + 1] - a_.in_off[static_cast<std::size_t>(v)]);
        std::int32_t d = static_cast<std::int32_t>(a_.off[v + 1] - a_.off[v]);
        if (a_.loop[v])  // only looped vertices need their out-edges counted
          for (EdgeId k = a_.off[v]; k < a_.off[v + 1]; ++k) d -= a_.tgt[k] == v;
        dout_[static_cast<std::size_t>(v)] = d;
      }
    });
    clk_.mark("partition: degrees");
    trim();
    clk_.mark("partition: trim");
    reach_giant();
    clk_.mark("partition: giant SCC (fw/bw reach)");
    trim();
    clk_.mark("partition: trim 2");
    tarjan_rest();
    clk_.mark("partition: Tarjan on the rest");
    return std::move(label_);
  }

 private:
  bool live(VertexId v) const { return label_[static_cast<std::size_t>(v)] < 0; }

  // Vertices without a live in-edge or out-edge are SCCs of their own; peel
  // them in rounds until none is left.
  void trim() {
    const int T = host_threads();
    Frontier next(T);
    parallel_chunks(n_, [&](int th, std::int64_t b, std::int64_t e) {
      for (std::int64_t v = b; v < e; ++v)
        if (live(static_cast<VertexId>(v)) && (din_[static_cast<std::size_t>(v)] == 0 || dout_[static_cast<std::size_t>(v)] == 0) &&
            claim(queued_[static_cast<std::size_t>(v)]))
          next.parts[static_cast<std::size_t>(th)].push_back(static_cast<std::int32_t>(v));
    });
    std::vector<std::int32_t> cur = next.take();
    while (!cur.empty()) {
      for_items(cur, [&](int, VertexId v) { label_[static_cast<std::size_t>(v)] = v; }, 1 << 16);
      for_items(cur, [&](int th, VertexId v) {
        auto& out = next.parts[static_cast<std::size_t>(th)];
        for (EdgeId k = a_.off[v]; k < a_.off[v + 1]; ++k) {
          const VertexId w = a_.tgt[k];
          if (w != v && live(w) && atomic_sub(din_[static_cast<std::size_t>(w)], 1) == 1 && claim(queued_[static_cast<std::size_t>(w)]))
            out.push_back(w);
        }
        for (EdgeId k = a_.in_off[static_cast<std::size_t>(v)]; k < a_.in_off[static_cast<std::size_t>(v) + 1]; ++k) {
          const VertexId p = a_.in_src[static_cast<std::size_t>(k)];
          if (live(p) && atomic_sub(dout_[static_cast<std::size_t>(p)], 1) == 1 && claim(queued_[static_cast<std::size_t>(p)]))
            out.push_back(p);
        }
      }, item_grain(n_));
      cur = next.take();
    }
  }

  // Forward and backward reachability from the live vertex of largest
  // din*dout; the intersection is its SCC (the giant SCC of a scale-free
  // graph).  Live set and visited sets are bitmaps (a few MB: they stay in
  // cache while the edge lists stream).
  void reach_giant() {
    std::int64_t best = -1;
    VertexId pivot = -1;
    {  // the first live vertex of largest din * dout (per-thread candidates over ascending ranges, merged in order)
      const int T = host_threads();
      std::vector<std::int64_t> tb(static_cast<std::size_t>(T), -1);
      std::vector<VertexId> tp(static_cast<std::size_t>(T), -1);
      parallel_chunks(n_, [&](int th, std::int64_t b, std::int64_t e) {
        std::int64_t lb = -1;
        VertexId lp = -1;
        for (std::int64_t vv = b; vv < e; ++vv) {
          const VertexId v = static_cast<VertexId>(vv);
          if (!live(v)) continue;
          const std::int64_t s = static_cast<std::int64_t>(din_[static_cast<std::size_t>(v)]) * dout_[static_cast<std::size_t>(v)];
          if (s > lb) lb = s, lp = v;
        }
        tb[static_cast<std::size_t>(th)] = lb;
        tp[static_cast<std::size_t>(th)] = lp;
      });
      for (int t = 0; t < T; ++t)
        if (tb[static_cast<std::size_t>(t)] > best) best = tb[static_cast<std::size_t>(t)], pivot = tp[static_cast<std::size_t>(t)];
    }
    // no hub (a deep DAG of small components, planted SCCs): Tarjan alone
    if (pivot < 0 || best < kMinHubDegreeProduct) return;
    const std::size_t nn = static_cast<std::size_t>(n_);
    Bits alive(nn), fw(nn), bw(nn);
    parallel_chunks((n_ + 63) / 64, [&](int, std::int64_t b, std::int64_t e) {
      for (std::int64_t wd = b; wd < e; ++wd) {
        std::uint64_t x = 0;
        for (std::int64_t v = wd * 64, k = 0; k < 64 && v < n_; ++v, ++k) x |= static_cast<std::uint64_t>(live(static_cast<VertexId>(v))) << k;
        alive.w[static_cast<std::size_t>(wd)] = x;
      }
    });
    // a pivot whose reach needs more than kMaxReachLevels BFS levels sits in a
    // deep DAG of small components (config 4), not in a giant SCC: leave it
    // to Tarjan (the result is the same, only the order of work changes)
    // The two searches share nothing but read-only inputs and are bound by
    // memory latency, not by the cores: they run side by side (the backward one
    // on its own thread; its parallel loops find the pool busy and spawn theirs).
    // LR_REACH_SERIAL=1 runs them one after the other.
    bool fw_ok = false, bw_ok = false;
    if (std::getenv("LR_REACH_SERIAL") != nullptr) {
      fw_ok = bfs(pivot, alive, fw, false);
      bw_ok = fw_ok && bfs(pivot, alive, bw, true);
    } else {
      std::exception_ptr back_error;
      std::thread back([&] {
        try {
          bw_ok = bfs(pivot, alive, bw, true);
        } catch (...) {
          back_error = std::current_exception();
        }
      });
      try {
        fw_ok = bfs(pivot, alive, fw, false);
      } catch (...) {
        back.join();
        throw;
      }
      back.join();
      if (back_error) std::rethrow_exception(back_error);
    }
    if (!fw_ok || !bw_ok) return;
    giant_ = pivot;
    // the SCC's members leave the graph: recount live degrees without them
    parallel_chunks(n_, [&](int, std::int64_t b, std::int64_t e) {
      for (std::int64_t v = b; v < e; ++v)
        if (fw.get(static_cast<VertexId>(v)) && bw.get(static_cast<VertexId>(v))) {
          label_[static_cast<std::size_t>(v)] = pivot;
          alive.clear_atomic(static_cast<VertexId>(v));
        }
    });
    parallel_chunks(n_, [&](int, std::int64_t b, std::int64_t e) {
      for (std::int64_t vv = b; vv < e; ++vv) {
        const VertexId v = static_cast<VertexId>(vv);
        if (!alive.get(v)) continue;
        std::int32_t di = 0, dout = 0;
        for (EdgeId k = a_.off[v]; k < a_.off[v + 1]; ++k) dout += a_.tgt[k] != v && alive.get(a_.tgt[k]);
        for (EdgeId k = a_.in_off[static_cast<std::size_t>(v)]; k < a_.in_off[static_cast<std::size_t>(v) + 1]; ++k)
          di += alive.get(a_.in_src[static_cast<std::size_t>(k)]);
        din_[static_cast<std::size_t>(v)] = di;
        dout_[static_cast<std::size_t>(v)] = dout;
      }
    });
  }

  // Level-synchronous BFS over the live vertices, direction-optimising
  // (Beamer et al.): a large frontier switches to the bottom-up step, where
  // every unvisited vertex looks for one parent in the frontier and stops.
  static constexpr int kMaxReachLevels = 128;
  static constexpr std::int64_t kMinHubDegreeProduct = 1024;
  bool bfs(VertexId src, const Bits& alive, Bits& seen, bool backward) {
    const int T = host_threads();
    const EdgeId* fo = backward ? a_.in_off.data() : a_.off;  // search direction
    const VertexId* fa = backward ? a_.in_src.data() : a_.tgt;
    const EdgeId* ro = backward ? a_.off : a_.in_off.data();  // parents in the search direction
    const VertexId* ra = backward ? a_.tgt : a_.in_src.data();
    Frontier next(T);
    Bits in_front(static_cast<std::size_t>(n_));
    seen.set_atomic(src);
    std::vector<std::int32_t> cur{src};
    EdgeId unexplored = fo[n_] - fo[0];
    bool bottom_up = false;
    int levels = 0;
    while (!cur.empty()) {
      std::atomic<EdgeId> fe{0};
      for_items(cur, [&](int, VertexId v) { fe.fetch_add(fo[v + 1] - fo[v], std::memory_order_relaxed); }, item_grain(n_));
      if (!bottom_up && fe.load() > unexplored / 14) bottom_up = true;
      else if (bottom_up && static_cast<std::int64_t>(cur.size()) < n_ / 24) bottom_up = false;
      unexplored -= fe.load();
      if (bottom_up) {
        std::fill(in_front.w.begin(), in_front.w.end(), 0);
        for_items(cur, [&](int, VertexId v) { in_front.set_atomic(v); }, item_grain(n_));
        parallel_chunks(n_, [&](int th, std::int64_t b, std::int64_t e) {
          auto& out = next.parts[static_cast<std::size_t>(th)];
          for (std::int64_t ww = b; ww < e; ++ww) {
            const VertexId w = static_cast<VertexId>(ww);
            if (!alive.get(w) || seen.get(w)) continue;
            for (EdgeId k = ro[w]; k < ro[w + 1]; ++k)
              if (in_front.get(ra[k])) {
                seen.set_atomic(w);
                out.push_back(w);
                break;
              }
          }
        });
      } else {
        for_items(cur, [&](int th, VertexId v) {
          auto& out = next.parts[static_cast<std::size_t>(th)];
          for (EdgeId k = fo[v]; k < fo[v + 1]; ++k) {
            const VertexId w = fa[k];
            if (alive.get(w) && seen.set_atomic(w)) out.push_back(w);
          }
        }, item_grain(n_));
      }
      cur = next.take();
      if (++levels > kMaxReachLevels && !cur.empty()) return false;
    }
    return true;
  }

  // Tarjan's algorithm (SCC labels only) over the live vertices.
  void tarjan_rest() {
    const std::size_t nn = static_cast<std::size_t>(n_);
    uvector<std::int32_t> order = detail::filled<std::int32_t>(nn, -1), low(nn);  // low is set when a vertex opens
    std::vector<VertexId> pending;
    std::vector<std::pair<VertexId, EdgeId>> stack;
    std::int32_t clock = 0;
    for (VertexId s = 0; s < n_; ++s) {
      if (!live(s) || order[static_cast<std::size_t>(s)] >= 0) continue;
      auto open = [&](VertexId v) {
        order[static_cast<std::size_t>(v)] = low[static_cast<std::size_t>(v)] = clock++;
        pending.push_back(v);
        stack.emplace_back(v, a_.off[v]);
      };
      open(s);
      while (!stack.empty()) {
        auto& top = stack.back();
        const VertexId v = top.first;
        if (top.second < a_.off[v + 1]) {
          const VertexId w = a_.tgt[top.second++];
          if (w == v || !live(w)) continue;
          if (order[static_cast<std::size_t>(w)] < 0) open(w);
          else low[static_cast<std::size_t>(v)] = std::min(low[static_cast<std::size_t>(v)], low[static_cast<std::size_t>(w)]);
          continue;
        }
        stack.pop_back();
        if (!stack.empty()) {
          const VertexId p = stack.back().first;
          low[static_cast<std::size_t>(p)] = std::min(low[static_cast<std::size_t>(p)], low[static_cast<std::size_t>(v)]);
        }
        if (low[static_cast<std::size_t>(v)] != order[static_cast<std::size_t>(v)]) continue;
        VertexId m;
        do {
          m = pending.back();
          pending.pop_back();
          label_[static_cast<std::size_t>(m)] = v;  // leaves the live set
          low[static_cast<std::size_t>(m)] = n_;    // never lowers a later low
        } while (m != v);
      }
    }
  }

  VertexId n_;
  const Adjacency& a_;
  detail::PhaseClock& clk_;
 public:
  VertexId giant_ = -1;  // representative of the SCC found by reachability (-1: none)
 private:
  uvector<VertexId> label_;
  uvector<std::int32_t> din_, dout_;
  uvector<std::uint8_t> queued_;
};

// Disjoint sets over component indices (union by size, path halving).
struct Sets {
  uvector<std::int32_t> up;
  explicit Sets(std::int32_t k) : up(detail::filled<std::int32_t>(static_cast<std::size_t>(k), -1)) {}
  std::int32_t find(std::int32_t x) {
    while (up[static_cast<std::size_t>(x)] >= 0) {
      const std::int32_t p = up[static_cast<std::size_t>(x)];
      if (up[static_cast<std::size_t>(p)] >= 0) up[static_cast<std::size_t>(x)] = up[static_cast<std::size_t>(p)];
      x = p;
    }
    return x;
  }
  void unite(std::int32_t a, std::int32_t b) {
    a = find(a);
    b = find(b);
    if (a == b) return;
    if (up[static_cast<std::size_t>(a)] > up[static_cast<std::size_t>(b)]) std::swap(a, b);
    up[static_cast<std::size_t>(a)] += up[static_cast<std::size_t>(b)];
    up[static_cast<std::size_t>(b)] = a;
  }
};

constexpr std::int64_t kWideComponent = 1 << 14;  // members scanned in parallel above this
constexpr EdgeId kAhead = 16;                      // software prefetch distance on edge scans

Partition wavefront_partition(const Graph& g, bool absorb_cacs, PartitionStats* stats, detail::InEdges* keep_in) {
  const VertexId n = g.vertex_count();
  const std::size_t nn = static_cast<std::size_t>(n);
  Partition p;
  PartitionStats st;
  st.explore_edge_visits = g.edge_count();
  st.finish_calls = n;
  if (n == 0) {
    if (stats) *stats = st;
    if (keep_in) keep_in->off.assign(1, 0);
    return p;
  }
  detail::PhaseClock clk;
  Adjacency adj{g.offsets_data(), g.targets_data(), g.loop_data(), {}, {}};
  {
    uvector<EdgeId> ptr[1];
    uvector<VertexId> col[1];
    detail::bucket_csr<1>(
        n, n,
        [&](std::int64_t uu, auto&& sink) {
          const VertexId u = static_cast<VertexId>(uu);
          for (EdgeId k = adj.off[u]; k < adj.off[u + 1]; ++k)
            if (adj.tgt[k] != u) sink(0, adj.tgt[k], u);
        },
        ptr, col);
    adj.in_off = std::move(ptr[0]);
    adj.in_src = std::move(col[0]);
  }
  clk.mark("partition: in-edge transpose");
  const EdgeId m_all = adj.off[n], m_in = adj.in_off[nn];
  SccFinder finder(n, adj, clk);
  const uvector<VertexId> label = finder.run();
  const VertexId giant = finder.giant_;

  // dense component index per vertex (components numbered by representative)
  uvector<std::int32_t> cidx(nn + 1);
  cidx[nn] = 0;
  parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t v = b; v < e; ++v) cidx[static_cast<std::size_t>(v)] = label[static_cast<std::size_t>(v)] == v;
  });
  const std::int32_t K = detail::exclusive_scan_inplace(cidx.data(), static_cast<std::int64_t>(nn) + 1);
  uvector<std::int32_t> comp(nn);
  parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t v = b; v < e; ++v) comp[static_cast<std::size_t>(v)] = cidx[static_cast<std::size_t>(label[static_cast<std::size_t>(v)])];
  });
  uvector<std::int32_t>().swap(cidx);
  // edges that leave their SCC, one bit each (plan_internal.hpp): recorded by the
  // two scans below that look every edge's components up anyway
  uvector<std::uint64_t> cross_out(static_cast<std::size_t>((m_all + 63) / 64)), cross_in(static_cast<std::size_t>((m_in + 63) / 64));
  parallel_chunks(static_cast<std::int64_t>(cross_out.size()), [&](int, std::int64_t b, std::int64_t e) { std::fill(cross_out.begin() + b, cross_out.begin() + e, 0); });
  parallel_chunks(static_cast<std::int64_t>(cross_in.size()), [&](int, std::int64_t b, std::int64_t e) { std::fill(cross_in.begin() + b, cross_in.begin() + e, 0); });
  // members grouped by component (CSR), cross out-edge counts.  The giant
  // SCC (one component, a large share of the vertices) is counted per thread
  // instead of by atomics on one counter.
  const std::size_t KK = static_cast<std::size_t>(K);
  const std::int32_t cg = giant >= 0 ? comp[static_cast<std::size_t>(giant)] : -1;
  const int T = host_threads();
  uvector<std::int64_t> mptr = detail::filled<std::int64_t>(KK + 1, 0);
  uvector<std::int64_t> pending = detail::filled<std::int64_t>(KK, 0);
  std::vector<std::vector<VertexId>> gmem(static_cast<std::size_t>(T));
  std::vector<std::int64_t> gpend(static_cast<std::size_t>(T), 0);
  // Membership in the giant SCC as a bitmap (8 MB at 2^26 vertices: cache
  // resident, unlike comp[]): an edge with an end in the giant SCC is classified
  // without looking its components up -- both ends inside: not cross; one end
  // inside: cross, and the inside end's component is cg.  On a scale-free graph
  // that covers nearly every edge.
  Bits in_giant(cg >= 0 ? nn : 0);
  if (cg >= 0)
    parallel_chunks((n + 63) / 64, [&](int, std::int64_t b, std::int64_t e) {
      for (std::int64_t wd = b; wd < e; ++wd) {
        std::uint64_t x = 0;
        for (std::int64_t v = wd * 64, k = 0; k < 64 && v < n; ++v, ++k) x |= static_cast<std::uint64_t>(comp[static_cast<std::size_t>(v)] == cg) << k;
        in_giant.w[static_cast<std::size_t>(wd)] = x;
      }
    });
  parallel_chunks(n, [&](int th, std::int64_t b, std::int64_t e) {
    detail::CrossBits bits(cross_out.data());
    for (std::int64_t vv = b; vv < e; ++vv) {
      const VertexId v = static_cast<VertexId>(vv);
      const std::int32_t c = comp[static_cast<std::size_t>(v)];
      std::int64_t x = 0;
      const EdgeId k1 = adj.off[v + 1];
      if (cg >= 0) {
        if (c == cg) {  // its cross out-edges are found from their targets below
          gmem[static_cast<std::size_t>(th)].push_back(v);
          continue;
        }
        for (EdgeId k = adj.off[v]; k < k1; ++k) {
          const VertexId w = adj.tgt[k];
          if (in_giant.get(w) || comp[static_cast<std::size_t>(w)] != c) {
            ++x;
            bits.set(k);
          }
        }
      } else {
        for (EdgeId k = adj.off[v]; k < k1; ++k) {
          if (k + kAhead < m_all) __builtin_prefetch(&comp[static_cast<std::size_t>(adj.tgt[k + kAhead])]);
          if (comp[static_cast<std::size_t>(adj.tgt[k])] != c) {
            ++x;
            bits.set(k);
          }
        }
      }
      if (c == cg) {
        gmem[static_cast<std::size_t>(th)].push_back(v);
        gpend[static_cast<std::size_t>(th)] += x;
        continue;
      }
      std::atomic_ref<std::int64_t>(mptr[static_cast<std::size_t>(c)]).fetch_add(1, std::memory_order_relaxed);
      if (x) std::atomic_ref<std::int64_t>(pending[static_cast<std::size_t>(c)]).fetch_add(x, std::memory_order_relaxed);
    }
  });
  // The giant SCC's cross out-edges, found from their targets: only a vertex
  // outside it can receive one, and those hold a small share of the in-edges --
  // no pass over the giant's own out-edge lists.  The edge's place in its source's
  // (target-ascending) row, for the cross-edge bit, is a binary search.
  if (cg >= 0)
    parallel_chunks(n, [&](int th, std::int64_t b, std::int64_t e) {
      std::int64_t found = 0;
      for (std::int64_t ww = b; ww < e; ++ww) {
        const VertexId w = static_cast<VertexId>(ww);
        if (in_giant.get(w)) continue;
        for (EdgeId k = adj.in_off[static_cast<std::size_t>(w)]; k < adj.in_off[static_cast<std::size_t>(w) + 1]; ++k) {
          const VertexId src = adj.in_src[static_cast<std::size_t>(k)];
          if (!in_giant.get(src)) continue;
          ++found;
          const EdgeId pos = std::lower_bound(adj.tgt + adj.off[src], adj.tgt + adj.off[src + 1], w) - adj.tgt;
          __atomic_fetch_or(&cross_out[static_cast<std::size_t>(pos >> 6)], std::uint64_t{1} << (pos & 63), __ATOMIC_RELAXED);
        }
      }
      gpend[static_cast<std::size_t>(th)] += found;
    });
  if (cg >= 0) {
    mptr[static_cast<std::size_t>(cg)] = 0;
    for (int t = 0; t < T; ++t) {
      mptr[static_cast<std::size_t>(cg)] += static_cast<std::int64_t>(gmem[static_cast<std::size_t>(t)].size());
      pending[static_cast<std::size_t>(cg)] += gpend[static_cast<std::size_t>(t)];
    }
  }
  uvector<std::int32_t> csize(KK);
  parallel_chunks(K, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t c = b; c < e; ++c) csize[static_cast<std::size_t>(c)] = static_cast<std::int32_t>(mptr[static_cast<std::size_t>(c)]);
  });
  detail::exclusive_scan_inplace(mptr.data(), static_cast<std::int64_t>(KK) + 1);
  uvector<VertexId> members(nn);
  {
    uvector<std::int64_t> fill(KK);
    parallel_chunks(K, [&](int, std::int64_t b, std::int64_t e) { std::copy(mptr.begin() + b, mptr.begin() + e, fill.begin() + b); });
    parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
      for (std::int64_t v = b; v < e; ++v) {
        const std::int32_t c = comp[static_cast<std::size_t>(v)];
        if (c == cg) continue;
        const std::int64_t at = csize[static_cast<std::size_t>(c)] == 1
                                    ? fill[static_cast<std::size_t>(c)]
                                    : std::atomic_ref<std::int64_t>(fill[static_cast<std::size_t>(c)]).fetch_add(1, std::memory_order_relaxed);
        members[static_cast<std::size_t>(at)] = static_cast<VertexId>(v);
      }
    });
    if (cg >= 0) {
      std::int64_t at = mptr[static_cast<std::size_t>(cg)];
      for (auto& part : gmem) {
        std::copy(part.begin(), part.end(), members.begin() + at);
        at += static_cast<std::int64_t>(part.size());
        std::vector<VertexId>().swap(part);
      }
    }
  }

  clk.mark("partition: components, members");
  // 2. wavefronts from the sinks of the component DAG
  uvector<std::int32_t> level = detail::filled<std::int32_t>(KK, 0);
  std::vector<std::vector<std::pair<std::int32_t, std::int32_t>>> absorbs(static_cast<std::size_t>(T));
  std::vector<std::int64_t> scans(static_cast<std::size_t>(T), 0);
  Frontier next(T);
  parallel_chunks(K, [&](int th, std::int64_t b, std::int64_t e) {
    for (std::int64_t c = b; c < e; ++c)
      if (pending[static_cast<std::size_t>(c)] == 0) next.parts[static_cast<std::size_t>(th)].push_back(static_cast<std::int32_t>(c));
  });
  std::vector<std::int32_t> cur = next.take();
  auto max_successor = [&](std::int32_t c, std::int64_t m0, std::int64_t m1) {
    std::int32_t hi = 0;
    for (std::int64_t i = m0; i < m1; ++i) {
      const VertexId u = members[static_cast<std::size_t>(i)];
      detail::for_cross_bits(cross_out.data(), adj.off[u], adj.off[u + 1], [&](EdgeId k) {
        hi = std::max(hi, level[static_cast<std::size_t>(comp[static_cast<std::size_t>(adj.tgt[k])])]);
      });
    }
    (void)c;
    return hi;
  };
  auto release = [&](int th, std::int32_t c, std::int64_t m0, std::int64_t m1) {
    auto& out = next.parts[static_cast<std::size_t>(th)];
    detail::CrossBits bits(cross_in.data());
    for (std::int64_t i = m0; i < m1; ++i) {
      const VertexId u = members[static_cast<std::size_t>(i)];
      const EdgeId k1 = adj.in_off[static_cast<std::size_t>(u) + 1];
      if (cg >= 0) {
        const bool ug = c == cg;
        for (EdgeId k = adj.in_off[static_cast<std::size_t>(u)]; k < k1; ++k) {
          const VertexId src = adj.in_src[static_cast<std::size_t>(k)];
          const bool sg = in_giant.get(src);
          if (ug && sg) continue;  // inside the giant SCC
          const std::int32_t cp = sg ? cg : comp[static_cast<std::size_t>(src)];
          if (cp == c) continue;
          bits.set(k);
          if (atomic_sub(pending[static_cast<std::size_t>(cp)], std::int64_t{1}) == 1) out.push_back(cp);
        }
        continue;
      }
      for (EdgeId k = adj.in_off[static_cast<std::size_t>(u)]; k < k1; ++k) {
        if (k + kAhead < m_in) __builtin_prefetch(&comp[static_cast<std::size_t>(adj.in_src[static_cast<std::size_t>(k + kAhead)])]);
        const std::int32_t cp = comp[static_cast<std::size_t>(adj.in_src[static_cast<std::size_t>(k)])];
        if (cp == c) continue;
        bits.set(k);
        if (atomic_sub(pending[static_cast<std::size_t>(cp)], std::int64_t{1}) == 1) out.push_back(cp);
      }
    }
  };
  // decide one component whose successors are all decided
  auto decide = [&](int th, std::int32_t c, std::int32_t hi) {
    const std::int32_t l0 = hi + 1;
    level[static_cast<std::size_t>(c)] = l0;
    if (csize[static_cast<std::size_t>(c)] != 1 || !absorb_cacs) return;
    const VertexId v = members[static_cast<std::size_t>(mptr[static_cast<std::size_t>(c)])];
    auto& mine = absorbs[static_cast<std::size_t>(th)];
    const std::size_t mark = mine.size();
    std::int64_t scanned = 0;
    bool veto = false;
    for (EdgeId k = adj.off[v]; k < adj.off[v + 1]; ++k) {
      ++scanned;
      const VertexId w = adj.tgt[k];
      if (w == v) continue;
      const std::int32_t cw = comp[static_cast<std::size_t>(w)];
      if (level[static_cast<std::size_t>(cw)] != l0 - 1) continue;
      if (csize[static_cast<std::size_t>(cw)] > 1) {
        veto = true;
        break;
      }
      mine.emplace_back(c, cw);
    }
    scans[static_cast<std::size_t>(th)] += scanned;
    if (veto) mine.resize(mark);
    else if (mine.size() > mark) level[static_cast<std::size_t>(c)] = l0 - 1;
  };
  long long n_waves = 0, n_items = 0;
  while (!cur.empty()) {
    ++n_waves;
    n_items += static_cast<long long>(cur.size());
    // the few components with many members (the giant SCC) are scanned member-parallel;
    // the rest one component per item (the item loops below skip the wide ones)
    auto is_wide = [&](std::int32_t c) { return csize[static_cast<std::size_t>(c)] > kWideComponent; };
    const std::vector<std::int32_t>& narrow = cur;
    std::vector<std::int32_t> wide;
    {
      std::vector<std::vector<std::int32_t>> found(static_cast<std::size_t>(T));
      for_items(cur, [&](int th, std::int32_t c) { if (is_wide(c)) found[static_cast<std::size_t>(th)].push_back(c); }, 1 << 16);
      for (const auto& f : found) wide.insert(wide.end(), f.begin(), f.end());
      std::sort(wide.begin(), wide.end());
    }
    for (const std::int32_t c : wide) {  // the giant SCC: members in parallel
      const std::int64_t m0 = mptr[static_cast<std::size_t>(c)], m1 = mptr[static_cast<std::size_t>(c) + 1];
      std::vector<std::int32_t> his(static_cast<std::size_t>(T), 0);
      parallel_chunks(m1 - m0, [&](int th, std::int64_t b, std::int64_t e) {
        his[static_cast<std::size_t>(th)] = std::max(his[static_cast<std::size_t>(th)], max_successor(c, m0 + b, m0 + e));
      });
      decide(0, c, *std::max_element(his.begin(), his.end()));
    }
    for_items(narrow, [&](int th, std::int32_t c) {
      if (is_wide(c)) return;
      decide(th, c, max_successor(c, mptr[static_cast<std::size_t>(c)], mptr[static_cast<std::size_t>(c) + 1]));
    }, item_grain(n));
    for (const std::int32_t c : wide) {
      if (c == cg) {
        // The giant SCC's cross in-edges, found from their sources: only the
        // vertices outside it can hold one, and those carry a small share of the
        // edges -- no pass over the giant's own in-edge lists.  The edge's place in
        // its target's (source-ascending) in-list, for the cross-edge bit, is a
        // binary search.
        parallel_chunks(n, [&](int th, std::int64_t b, std::int64_t e) {
          auto& out = next.parts[static_cast<std::size_t>(th)];
          for (std::int64_t pp = b; pp < e; ++pp) {
            const VertexId pv = static_cast<VertexId>(pp);
            if (in_giant.get(pv)) continue;
            std::int64_t cnt = 0;
            for (EdgeId k = adj.off[pv]; k < adj.off[pv + 1]; ++k) {
              const VertexId w = adj.tgt[k];
              if (!in_giant.get(w)) continue;
              ++cnt;
              const VertexId* lo = adj.in_src.data() + adj.in_off[static_cast<std::size_t>(w)];
              const VertexId* hi = adj.in_src.data() + adj.in_off[static_cast<std::size_t>(w) + 1];
              const EdgeId pos = std::lower_bound(lo, hi, pv) - adj.in_src.data();
              __atomic_fetch_or(&cross_in[static_cast<std::size_t>(pos >> 6)], std::uint64_t{1} << (pos & 63), __ATOMIC_RELAXED);
            }
            if (cnt == 0) continue;
            const std::int32_t cp = comp[static_cast<std::size_t>(pv)];
            if (atomic_sub(pending[static_cast<std::size_t>(cp)], cnt) == cnt) out.push_back(cp);
          }
        });
        continue;
      }
      const std::int64_t m0 = mptr[static_cast<std::size_t>(c)], m1 = mptr[static_cast<std::size_t>(c) + 1];
      parallel_chunks(m1 - m0, [&](int th, std::int64_t b, std::int64_t e) { release(th, c, m0 + b, m0 + e); });
    }
    for_items(narrow, [&](int th, std::int32_t c) {
      if (is_wide(c)) return;
      release(th, c, mptr[static_cast<std::size_t>(c)], mptr[static_cast<std::size_t>(c) + 1]);
    }, item_grain(n));
    cur = next.take();
  }
  for (const std::int64_t s : scans) st.merge_scan_edge_visits += s;

  if (clk.on) std::fprintf(stderr, "[plan] partition: %lld wavefronts, %lld components\n", n_waves, n_items);
  clk.mark("partition: level wavefronts");
  // 3. absorptions -> final components, ids by smallest member
  Sets sets(K);
  uvector<std::int32_t> root(KK);
  parallel_chunks(K, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t c = b; c < e; ++c) root[static_cast<std::size_t>(c)] = static_cast<std::int32_t>(c);
  });
  std::vector<std::int32_t> touched;  // only components in an absorption change root
  for (const auto& part : absorbs)
    for (const auto& [a, b] : part) {
      sets.unite(a, b);
      touched.push_back(a);
      touched.push_back(b);
    }
  for (const std::int32_t c : touched) root[static_cast<std::size_t>(c)] = sets.find(c);
  // Everything below walks the components, not the vertices: a component's
  // smallest member, the smallest member of its final component (`first`), the
  // final id, its size; the vertices then take their id with one lookup each.
  uvector<VertexId> first = detail::filled<VertexId>(KK, n), minv(KK);
  parallel_chunks(K, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t c = b; c < e; ++c) {
      const std::int64_t m0 = mptr[static_cast<std::size_t>(c)], m1 = mptr[static_cast<std::size_t>(c) + 1];
      VertexId mn = members[static_cast<std::size_t>(m0)];
      for (std::int64_t i = m0 + 1; i < m1; ++i) mn = std::min(mn, members[static_cast<std::size_t>(i)]);
      minv[static_cast<std::size_t>(c)] = mn;
      std::atomic_ref<VertexId> f(first[static_cast<std::size_t>(root[static_cast<std::size_t>(c)])]);
      VertexId cur_min = f.load(std::memory_order_relaxed);
      while (mn < cur_min && !f.compare_exchange_weak(cur_min, mn, std::memory_order_relaxed)) {
      }
    }
  }, 1 << 12);
  uvector<VertexId> id_at = detail::filled<VertexId>(nn + 1, 0);  // id_at[v] = number of components first seen before v
  parallel_chunks(K, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t c = b; c < e; ++c)
      if (minv[static_cast<std::size_t>(c)] == first[static_cast<std::size_t>(root[static_cast<std::size_t>(c)])])
        id_at[static_cast<std::size_t>(minv[static_cast<std::size_t>(c)])] = 1;
  }, 1 << 12);
  const VertexId k = detail::exclusive_scan_inplace(id_at.data(), static_cast<std::int64_t>(nn) + 1);
  p.comp_of.resize(nn);
  p.kinds.resize(static_cast<std::size_t>(k));
  p.levels.resize(static_cast<std::size_t>(k));
  p.sizes.assign(static_cast<std::size_t>(k), 0);
  uvector<VertexId> fid(KK);  // final id of every SCC-level component
  parallel_chunks(K, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t c = b; c < e; ++c) {
      const VertexId f = first[static_cast<std::size_t>(root[static_cast<std::size_t>(c)])];
      const VertexId id = id_at[static_cast<std::size_t>(f)];
      fid[static_cast<std::size_t>(c)] = id;
      std::atomic_ref<VertexId>(p.sizes[static_cast<std::size_t>(id)]).fetch_add(csize[static_cast<std::size_t>(c)], std::memory_order_relaxed);
      if (minv[static_cast<std::size_t>(c)] == f) {  // the component of the final component's first vertex
        p.kinds[static_cast<std::size_t>(id)] = csize[static_cast<std::size_t>(c)] > 1 ? ComponentKind::Scc : ComponentKind::Cac;
        p.levels[static_cast<std::size_t>(id)] = level[static_cast<std::size_t>(c)];
      }
    }
  }, 1 << 12);
  parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t v = b; v < e; ++v)
      p.comp_of[static_cast<std::size_t>(v)] = fid[static_cast<std::size_t>(comp[static_cast<std::size_t>(v)])];
  });
  {  // shift the lowest level to 0
    const int T2 = host_threads();
    std::vector<std::int32_t> los(static_cast<std::size_t>(T2), INT32_MAX), his(static_cast<std::size_t>(T2), INT32_MIN);
    parallel_chunks(k, [&](int th, std::int64_t b, std::int64_t e) {
      const auto [mn, mx] = std::minmax_element(p.levels.begin() + b, p.levels.begin() + e);
      los[static_cast<std::size_t>(th)] = std::min(los[static_cast<std::size_t>(th)], *mn);
      his[static_cast<std::size_t>(th)] = std::max(his[static_cast<std::size_t>(th)], *mx);
    });
    const std::int32_t lo = *std::min_element(los.begin(), los.end());
    parallel_chunks(k, [&](int, std::int64_t b, std::int64_t e) {
      for (std::int64_t i = b; i < e; ++i) p.levels[static_cast<std::size_t>(i)] -= lo;
    });
    p.max_level = *std::max_element(his.begin(), his.end()) - lo;
  }
  clk.mark("partition: unions + assemble");
  if (stats) *stats = st;
  if (keep_in) {
    keep_in->off = std::move(adj.in_off);
    keep_in->src = std::move(adj.in_src);
    keep_in->cross_out = std::move(cross_out);
    keep_in->cross_in = std::move(cross_in);
  }
  return p;
}

}  // namespace

Partition find_components(const Graph& g, PartitionStats* stats) { return wavefront_partition(g, true, stats, nullptr); }

Partition find_components_scc_only(const Graph& g) { return wavefront_partition(g, false, nullptr, nullptr); }

namespace detail {
Partition find_components_with_in_edges(const Graph& g, PartitionStats* stats, InEdges& in) {
  return wavefront_partition(g, true, stats, &in);
}
}  // namespace detail

// The partition in a form independent of id numbering: components as sorted
// member lists with kind and level, ordered (partition.hpp:56-66).
std::vector<CanonicalComponent> canonical_components(const Partition& p) {
  const std::size_t k = p.component_count();
  std::vector<std::size_t> at(k + 1, 0);
  for (const VertexId c : p.comp_of) ++at[static_cast<std::size_t>(c) + 1];
  for (std::size_t c = 0; c < k; ++c) at[c + 1] += at[c];
  std::vector<CanonicalComponent> cs(k);
  for (std::size_t c = 0; c < k; ++c) {
    cs[c].members.reserve(at[c + 1] - at[c]);
    cs[c].kind = p.kinds[c];
    cs[c].level = p.levels[c];
  }
  for (std::size_t v = 0; v < p.comp_of.size(); ++v)  // ascending v: member lists come out sorted
    cs[static_cast<std::size_t>(p.comp_of[v])].members.push_back(static_cast<VertexId>(v));
  std::sort(cs.begin(), cs.end());
  return cs;
}

std::vector<std::uint8_t> big_scc_flags(const Partition& p) {
  std::vector<std::uint8_t> f(p.comp_of.size());
  std::transform(p.comp_of.begin(), p.comp_of.end(), f.begin(),
                 [&](VertexId c) { return static_cast<std::uint8_t>(p.kinds[static_cast<std::size_t>(c)] == ComponentKind::Scc); });
  return f;
}

PartitionCensus census(const Partition& p) {
  PartitionCensus c;
  c.components = static_cast<std::int64_t>(p.component_count());
  c.max_level = p.max_level;
  c.level_count = p.max_level + 1;
  c.components_per_level.assign(static_cast<std::size_t>(p.max_level + 1), 0);
  std::vector<std::int64_t> bins(33, 0);  // sizes in (2^(b-1), 2^b]
  VertexId largest = 0;
  for (std::size_t i = 0; i < p.component_count(); ++i) {
    const bool scc = p.kinds[i] == ComponentKind::Scc;
    c.scc_components += scc;
    c.cac_components += !scc;
    c.singleton_cacs += !scc && p.sizes[i] == 1;
    ++c.components_per_level[static_cast<std::size_t>(p.levels[i])];
    if (p.sizes[i] > largest) {  // first component of the largest size decides the kind
      largest = p.sizes[i];
      c.largest_kind = p.kinds[i];
    }
    const auto s = static_cast<std::uint32_t>(p.sizes[i]);
    ++bins[static_cast<std::size_t>(s <= 1 ? 0 : 32 - __builtin_clz(s - 1))];
  }
  c.largest_component = largest;
  std::size_t top = bins.size();
  while (top > 0 && bins[top - 1] == 0) --top;
  for (std::size_t b = 0; b < top; ++b) c.size_histogram.emplace_back(VertexId{1} << b, bins[b]);
  return c;
}

}  // namespace b200
}  // namespace levelrank
