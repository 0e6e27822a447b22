// Seeded synthetic inputs for the BASELINE.json configs (DESIGN.md "Synthetic
// inputs").  Every random draw is a splitmix64 output addressed by
// (seed, stream, index), so generation is embarrassingly parallel and the
// result does not depend on the thread count.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <vector>

#include "levelrank/graph.hpp"
#include "parallel.hpp"

namespace levelrank {
inline namespace b200 {
namespace gen {

inline std::uint64_t mix(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
// i-th splitmix64 output of a stream keyed by (seed, stream)
inline std::uint64_t draw(std::uint64_t seed, std::uint64_t stream, std::uint64_t i) {
  const std::uint64_t key = mix(seed * 0x9E3779B97F4A7C15ULL + (stream + 1) * 0xD1B54A32D192ED03ULL);
  return mix(key + (i + 1) * 0x9E3779B97F4A7C15ULL);
}
inline double unit(std::uint64_t x) { return static_cast<double>(x >> 11) * 0x1.0p-53; }
// uniform integer in [0, n) (multiply-shift; bias < n / 2^64)
inline std::uint64_t below(std::uint64_t x, std::uint64_t n) {
  return static_cast<std::uint64_t>((static_cast<unsigned __int128>(x) * n) >> 64);
}

// R-MAT (Chakrabarti et al.) edge i: `scale` quadrant choices, two 32-bit
// uniforms per draw; self-loops are dropped here, duplicates by from_edges.
Graph rmat(std::int32_t scale, std::int64_t edge_factor, double a, double b, double c, std::uint64_t seed) {
  if (scale < 1 || scale > 30 || edge_factor < 1) throw std::invalid_argument("bad R-MAT size");
  const std::int64_t n = std::int64_t{1} << scale;
  const std::int64_t m = edge_factor << scale;
  const double ab = a + b, abc = a + b + c;
  const std::uint32_t ta = static_cast<std::uint32_t>(std::ldexp(a, 32) < 4294967295.0 ? std::ldexp(a, 32) : 4294967295.0);
  const std::uint32_t tab = static_cast<std::uint32_t>(std::min(std::ldexp(ab, 32), 4294967295.0));
  const std::uint32_t tabc = static_cast<std::uint32_t>(std::min(std::ldexp(abc, 32), 4294967295.0));
  const int per_edge = (scale + 1) / 2;
  const int T = host_threads();
  std::vector<std::int64_t> kept(static_cast<std::size_t>(T) + 1, 0);
  auto make = [&](std::int64_t i, VertexId& u, VertexId& v) {
    std::uint32_t su = 0, sv = 0;
    for (int l = 0; l < scale; ++l) {
      const std::uint64_t r = draw(seed, 1, static_cast<std::uint64_t>(i) * per_edge + l / 2);
      const std::uint32_t x = static_cast<std::uint32_t>((l & 1) ? (r >> 32) : r);
      const std::uint32_t bu = x >= tab, bv = (x >= ta && x < tab) || x >= tabc;
      su = (su << 1) | bu;
      sv = (sv << 1) | bv;
    }
    u = static_cast<VertexId>(su);
    v = static_cast<VertexId>(sv);
  };
  std::vector<std::int64_t> chunk_begin(static_cast<std::size_t>(T) + 1);
  for (int t = 0; t <= T; ++t) chunk_begin[static_cast<std::size_t>(t)] = m * t / T;
  // one pass: each thread keeps its chunk's non-loop edges, then the chunks
  // are concatenated in order (output independent of the thread count)
  std::vector<std::vector<VertexId>> ts(static_cast<std::size_t>(T)), td(static_cast<std::size_t>(T));
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      const std::int64_t b0 = chunk_begin[static_cast<std::size_t>(t)], b1 = chunk_begin[static_cast<std::size_t>(t) + 1];
      auto& S = ts[static_cast<std::size_t>(t)];
      auto& D = td[static_cast<std::size_t>(t)];
      S.reserve(static_cast<std::size_t>(b1 - b0));
      D.reserve(static_cast<std::size_t>(b1 - b0));
      for (std::int64_t i = b0; i < b1; ++i) {
        VertexId u, v;
        make(i, u, v);
        if (u == v) continue;
        S.push_back(u);
        D.push_back(v);
      }
      kept[static_cast<std::size_t>(t) + 1] = static_cast<std::int64_t>(S.size());
    });
  for (auto& th : pool) th.join();
  for (int t = 0; t < T; ++t) kept[static_cast<std::size_t>(t) + 1] += kept[static_cast<std::size_t>(t)];
  std::vector<VertexId> src(static_cast<std::size_t>(kept[static_cast<std::size_t>(T)])), dst(src.size());
  pool.clear();
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      auto& S = ts[static_cast<std::size_t>(t)];
      auto& D = td[static_cast<std::size_t>(t)];
      std::copy(S.begin(), S.end(), src.begin() + kept[static_cast<std::size_t>(t)]);
      std::copy(D.begin(), D.end(), dst.begin() + kept[static_cast<std::size_t>(t)]);
      std::vector<VertexId>().swap(S);
      std::vector<VertexId>().swap(D);
    });
  for (auto& th : pool) th.join();
  return Graph::from_edge_arrays(static_cast<VertexId>(n), src.data(), dst.data(), static_cast<EdgeId>(src.size()));
}

// Every vertex independently (probability p) loses all its out-edges.
Graph dangle(const Graph& g, double p, std::uint64_t seed) {
  const VertexId n = g.vertex_count();
  const std::size_t nn = static_cast<std::size_t>(n);
  std::vector<EdgeId> off(nn + 1, 0);
  std::vector<std::uint8_t> drop(nn);
  detail::parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t v = b; v < e; ++v) {
      drop[static_cast<std::size_t>(v)] = unit(draw(seed, 2, static_cast<std::uint64_t>(v))) < p;
      off[static_cast<std::size_t>(v)] = drop[static_cast<std::size_t>(v)] ? 0 : g.out_degree(static_cast<VertexId>(v));
    }
  });
  const EdgeId m = detail::exclusive_scan_inplace(off.data(), static_cast<std::int64_t>(nn) + 1);
  std::vector<VertexId> tgt(static_cast<std::size_t>(m));
  detail::parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t v = b; v < e; ++v) {
      if (drop[static_cast<std::size_t>(v)]) continue;
      const auto row = g.out_neighbors(static_cast<VertexId>(v));
      std::copy(row.begin(), row.end(), tgt.begin() + off[static_cast<std::size_t>(v)]);
    }
  });
  return Graph::from_csr(n, std::move(off), std::move(tgt), g.loop_policy());
}

// Planted components (config 1): n_scc SCCs (Hamiltonian cycle + ER chords)
// with sizes U[scc_min, scc_max] rescaled to `budget` vertices in total, the
// remaining vertices as random out-trees, `inter_edges` edges from lower to
// higher component index, a `dangling_fraction` of vertices (tree leaves)
// kept without out-edges.
Graph planted(VertexId n, std::int32_t n_scc, std::int32_t smin, std::int32_t smax, std::int64_t budget,
              double out_degree, std::int64_t inter_edges, double dangling_fraction, std::uint64_t seed) {
  std::uint64_t ctr = 0;
  auto next = [&](std::uint64_t stream) { return draw(seed, stream, ctr++); };
  std::vector<std::int64_t> size(static_cast<std::size_t>(n_scc));
  std::int64_t total = 0;
  for (auto& s : size) {
    s = smin + static_cast<std::int64_t>(below(next(10), static_cast<std::uint64_t>(smax - smin + 1)));
    total += s;
  }
  if (budget > 0 && total > budget)
    for (auto& s : size) s = std::max<std::int64_t>(smin, s * budget / total);
  total = std::accumulate(size.begin(), size.end(), std::int64_t{0});
  if (total > n) throw std::invalid_argument("planted SCCs exceed the vertex count");
  // random vertex labelling
  std::vector<VertexId> perm(static_cast<std::size_t>(n));
  std::iota(perm.begin(), perm.end(), 0);
  for (VertexId i = n - 1; i > 0; --i) std::swap(perm[static_cast<std::size_t>(i)], perm[static_cast<std::size_t>(below(next(11), static_cast<std::uint64_t>(i) + 1))]);
  std::vector<VertexId> src, dst;
  auto edge = [&](VertexId u, VertexId v) {
    src.push_back(perm[static_cast<std::size_t>(u)]);
    dst.push_back(perm[static_cast<std::size_t>(v)]);
  };
  // components as contiguous id ranges (before labelling); comp index order random
  std::vector<std::pair<VertexId, VertexId>> comp;  // [begin, end)
  VertexId at = 0;
  for (const auto s : size) {
    const VertexId b = at;
    at += static_cast<VertexId>(s);
    for (VertexId v = b; v < at; ++v) edge(v, v + 1 < at ? v + 1 : b);
    const double p = (out_degree - 1.0) / static_cast<double>(s - 1);
    for (VertexId u = b; u < at; ++u)
      for (VertexId v = b; v < at; ++v)
        if (u != v && unit(next(12)) < p) edge(u, v);
    comp.emplace_back(b, at);
  }
  std::vector<std::uint8_t> has_out(static_cast<std::size_t>(n), 0), leaf_candidate(static_cast<std::size_t>(n), 0);
  for (VertexId v = 0; v < at; ++v) has_out[static_cast<std::size_t>(v)] = 1;
  // random recursive out-trees over the rest: root with prob 1/16
  VertexId root = at;
  for (VertexId v = at; v < n; ++v) {
    if (v == root || below(next(13), 16) == 0) {
      if (v != root) comp.emplace_back(root, v);
      root = v;
      continue;
    }
    const VertexId parent = root + static_cast<VertexId>(below(next(14), static_cast<std::uint64_t>(v - root)));
    edge(parent, v);
    has_out[static_cast<std::size_t>(parent)] = 1;
  }
  if (at < n) comp.emplace_back(root, n);
  const std::size_t K = comp.size();
  std::vector<std::int32_t> cidx(K);
  std::iota(cidx.begin(), cidx.end(), 0);
  for (std::size_t i = K - 1; i > 0; --i) std::swap(cidx[i], cidx[static_cast<std::size_t>(below(next(15), i + 1))]);
  std::vector<std::int32_t> comp_at_index(K);
  for (std::size_t c = 0; c < K; ++c) comp_at_index[static_cast<std::size_t>(cidx[c])] = static_cast<std::int32_t>(c);
  std::vector<std::int32_t> comp_of(static_cast<std::size_t>(n));
  for (std::size_t c = 0; c < K; ++c)
    for (VertexId v = comp[c].first; v < comp[c].second; ++v) comp_of[static_cast<std::size_t>(v)] = static_cast<std::int32_t>(c);
  // dangling set: a random `dangling_fraction` of n among vertices without out-edges
  std::vector<VertexId> leaves;
  for (VertexId v = 0; v < n; ++v)
    if (!has_out[static_cast<std::size_t>(v)]) leaves.push_back(v);
  for (std::size_t i = leaves.size(); i > 1; --i) std::swap(leaves[i - 1], leaves[static_cast<std::size_t>(below(next(16), i))]);
  const std::size_t keep_dangling = std::min(leaves.size(), static_cast<std::size_t>(dangling_fraction * n));
  std::vector<std::uint8_t> dangling(static_cast<std::size_t>(n), 0);
  for (std::size_t i = 0; i < keep_dangling; ++i) dangling[static_cast<std::size_t>(leaves[i])] = 1;
  auto inter_from = [&](VertexId u) -> bool {
    const std::int32_t ci = cidx[static_cast<std::size_t>(comp_of[static_cast<std::size_t>(u)])];
    if (static_cast<std::size_t>(ci) + 1 >= K) return false;
    const std::int32_t cj = ci + 1 + static_cast<std::int32_t>(below(next(17), K - static_cast<std::size_t>(ci) - 1));
    const auto& [b, e] = comp[static_cast<std::size_t>(comp_at_index[static_cast<std::size_t>(cj)])];
    edge(u, b + static_cast<VertexId>(below(next(18), static_cast<std::uint64_t>(e - b))));
    return true;
  };
  std::int64_t used = 0;
  for (VertexId v = 0; v < n && used < inter_edges; ++v)
    if (!has_out[static_cast<std::size_t>(v)] && !dangling[static_cast<std::size_t>(v)]) used += inter_from(v);
  while (used < inter_edges) {
    const VertexId u = static_cast<VertexId>(below(next(19), static_cast<std::uint64_t>(n)));
    if (dangling[static_cast<std::size_t>(u)]) continue;
    used += inter_from(u) ? 1 : 0;
    if (K < 2) break;
  }
  return Graph::from_edge_arrays(n, src.data(), dst.data(), static_cast<EdgeId>(src.size()));
}

// Deep DAG of components (config 4): `levels` construction levels of `width`
// vertices, filled alternately with SCCs (size U[smin,smax], cycle + chords
// at `scc_out_degree`) and out-trees (size U[smin,smax], branching
// U[bmin,bmax]); every vertex sends inter-component edges (mean
// `inter_out_degree`) to uniform vertices of construction level + U[1,reach].
Graph deep_dag(std::int32_t levels, std::int32_t width, std::int32_t smin, std::int32_t smax, double scc_out_degree,
               std::int32_t bmin, std::int32_t bmax, double inter_out_degree, std::int32_t reach, std::uint64_t seed) {
  const std::int64_t n64 = static_cast<std::int64_t>(levels) * width;
  if (n64 > kMaxVertexId) throw std::invalid_argument("deep DAG too large");
  const VertexId n = static_cast<VertexId>(n64);
  const int T = host_threads();
  std::vector<std::vector<VertexId>> ts(static_cast<std::size_t>(T)), td(static_cast<std::size_t>(T));
  std::atomic<std::int32_t> next_level{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      auto& S = ts[static_cast<std::size_t>(t)];
      auto& D = td[static_cast<std::size_t>(t)];
      for (;;) {
        const std::int32_t lv = next_level.fetch_add(1);
        if (lv >= levels) return;
        std::uint64_t ctr = 0;
        auto rnd = [&](std::uint64_t stream) { return draw(seed, static_cast<std::uint64_t>(lv) * 64 + stream, ctr++); };
        const VertexId base = static_cast<VertexId>(static_cast<std::int64_t>(lv) * width);
        VertexId at = 0;
        bool scc = true;
        while (at < width) {
          const VertexId sz = std::min<VertexId>(width - at, smin + static_cast<VertexId>(below(rnd(1), static_cast<std::uint64_t>(smax - smin + 1))));
          const VertexId b = base + at, e = b + sz;
          if (scc && sz >= 2) {
            for (VertexId v = b; v < e; ++v) {
              S.push_back(v);
              D.push_back(v + 1 < e ? v + 1 : b);
            }
            const double extra = scc_out_degree - 1.0;
            for (VertexId v = b; v < e; ++v) {
              const std::int32_t k = static_cast<std::int32_t>(extra) + (unit(rnd(2)) < extra - std::floor(extra));
              for (std::int32_t j = 0; j < k; ++j) {
                VertexId w = b + static_cast<VertexId>(below(rnd(3), static_cast<std::uint64_t>(sz - 1)));
                if (w >= v) ++w;
                S.push_back(v);
                D.push_back(w);
              }
            }
          } else {
            // BFS out-tree: node i gets U[bmin,bmax] children in order
            VertexId filled = 1;
            for (VertexId i = 0; i < sz && filled < sz; ++i) {
              const VertexId kids = bmin + static_cast<VertexId>(below(rnd(4), static_cast<std::uint64_t>(bmax - bmin + 1)));
              for (VertexId j = 0; j < kids && filled < sz; ++j, ++filled) {
                S.push_back(b + i);
                D.push_back(b + filled);
              }
            }
          }
          at += sz;
          scc = !scc;
        }
        const double mean = inter_out_degree;
        for (VertexId v = base; v < base + width; ++v) {
          const std::int32_t k = static_cast<std::int32_t>(mean) + (unit(rnd(5)) < mean - std::floor(mean));
          for (std::int32_t j = 0; j < k; ++j) {
            const std::int32_t tl = lv + 1 + static_cast<std::int32_t>(below(rnd(6), static_cast<std::uint64_t>(reach)));
            if (tl >= levels) continue;
            S.push_back(v);
            D.push_back(static_cast<VertexId>(static_cast<std::int64_t>(tl) * width) +
                        static_cast<VertexId>(below(rnd(7), static_cast<std::uint64_t>(width))));
          }
        }
      }
    });
  for (auto& th : pool) th.join();
  std::size_t m = 0;
  for (const auto& s : ts) m += s.size();
  std::vector<VertexId> src, dst;
  src.reserve(m);
  dst.reserve(m);
  for (int t = 0; t < T; ++t) {
    src.insert(src.end(), ts[static_cast<std::size_t>(t)].begin(), ts[static_cast<std::size_t>(t)].end());
    dst.insert(dst.end(), td[static_cast<std::size_t>(t)].begin(), td[static_cast<std::size_t>(t)].end());
    ts[static_cast<std::size_t>(t)] = {};
    td[static_cast<std::size_t>(t)] = {};
  }
  return Graph::from_edge_arrays(n, src.data(), dst.data(), static_cast<EdgeId>(src.size()));
}

}  // namespace gen
}  // namespace b200
}  // namespace levelrank
