// Graph core: multi-threaded CSR build with Graph::from_edges semantics
// (proj/src/graph.cpp:14-36: range check, dedup, sorted rows, loop flags).
// The edge-list reader is in ingest.cpp.
#include "levelrank/graph.hpp"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <stdexcept>
#include <thread>

#include "parallel.hpp"

namespace levelrank {
inline namespace b200 {

int host_threads() {
  static const int t = [] {
    if (const char* e = std::getenv("LR_THREADS")) {
      const int v = std::atoi(e);
      if (v > 0) return v;
    }
    const unsigned h = std::thread::hardware_concurrency();
    return h ? static_cast<int>(std::min(h, 256u)) : 1;
  }();
  return t;
}

Graph Graph::from_edges(VertexId n, std::vector<std::pair<VertexId, VertexId>> edges,
                        LoopPolicy policy) {
  const EdgeId m = static_cast<EdgeId>(edges.size());
  std::vector<VertexId> src(static_cast<std::size_t>(m)), dst(static_cast<std::size_t>(m));
  detail::parallel_chunks(m, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t i = b; i < e; ++i) {
      src[static_cast<std::size_t>(i)] = edges[static_cast<std::size_t>(i)].first;
      dst[static_cast<std::size_t>(i)] = edges[static_cast<std::size_t>(i)].second;
    }
  });
  edges = {};
  return from_edge_arrays(n, src.data(), dst.data(), m, policy);
}

Graph Graph::from_edge_arrays(VertexId n, const VertexId* src, const VertexId* dst, EdgeId m,
                              LoopPolicy policy) {
  if (n < 0) throw std::invalid_argument("vertex count must be non-negative");
  std::atomic<bool> bad{false};
  detail::parallel_chunks(m, [&](int, std::int64_t b, std::int64_t e) {
    bool local = false;
    for (std::int64_t i = b; i < e; ++i)
      local |= src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n;
    if (local) bad = true;
  });
  if (bad) throw std::invalid_argument("edge endpoint out of range");

  const std::size_t nn = static_cast<std::size_t>(n);
  // rows by source: atomic-free stable bucketed transpose of the edge list
  std::vector<EdgeId> offs[1];
  std::vector<VertexId> cols[1];
  detail::bucket_csr<1>(
      m, n, [&](std::int64_t i, auto&& sink) { sink(0, src[i], dst[i]); }, offs, cols);
  std::vector<EdgeId> off = std::move(offs[0]);
  std::vector<VertexId> tmp = std::move(cols[0]);
  std::vector<EdgeId> deg(nn + 1, 0);
  detail::parallel_dynamic(n, 4096, [&](std::int64_t b, std::int64_t e) {
    for (std::int64_t u = b; u < e; ++u) {
      VertexId* row = tmp.data() + off[static_cast<std::size_t>(u)];
      VertexId* end = tmp.data() + off[static_cast<std::size_t>(u) + 1];
      std::sort(row, end);
      deg[static_cast<std::size_t>(u)] = std::unique(row, end) - row;
    }
  });
  Graph g;
  g.n_ = n;
  g.policy_ = policy;
  const EdgeId total = detail::exclusive_scan_inplace(deg.data(), static_cast<std::int64_t>(nn) + 1);
  if (total == m) {
    g.targets_ = std::move(tmp);
    g.offsets_ = std::move(off);
  } else {
    g.targets_.resize(static_cast<std::size_t>(total));
    detail::parallel_dynamic(n, 4096, [&](std::int64_t b, std::int64_t e) {
      for (std::int64_t u = b; u < e; ++u) {
        const std::size_t su = static_cast<std::size_t>(u);
        std::copy(tmp.data() + off[su], tmp.data() + off[su] + (deg[su + 1] - deg[su]),
                  g.targets_.data() + deg[su]);
      }
    });
    g.offsets_ = std::move(deg);
  }
  g.has_loop_.assign(nn, 0);
  detail::parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t u = b; u < e; ++u) {
      const auto row = g.out_neighbors(static_cast<VertexId>(u));
      g.has_loop_[static_cast<std::size_t>(u)] =
          std::binary_search(row.begin(), row.end(), static_cast<VertexId>(u)) ? 1 : 0;
    }
  });
  return g;
}

Graph Graph::from_csr(VertexId n, std::vector<EdgeId> offsets, std::vector<VertexId> targets,
                      LoopPolicy policy) {
  const std::size_t nn = static_cast<std::size_t>(n);
  if (n < 0 || offsets.size() != nn + 1 || offsets[0] != 0 ||
      offsets[nn] != static_cast<EdgeId>(targets.size()))
    throw std::invalid_argument("malformed CSR offsets");
  std::atomic<bool> bad{false};
  Graph g;
  g.n_ = n;
  g.policy_ = policy;
  g.offsets_ = std::move(offsets);
  g.targets_ = std::move(targets);
  g.has_loop_.assign(nn, 0);
  detail::parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) {
    bool local = false;
    for (std::int64_t u = b; u < e; ++u) {
      const EdgeId lo = g.offsets_[static_cast<std::size_t>(u)], hi = g.offsets_[static_cast<std::size_t>(u) + 1];
      if (hi < lo) {
        local = true;
        continue;
      }
      for (EdgeId k = lo; k < hi; ++k) {
        const VertexId v = g.targets_[static_cast<std::size_t>(k)];
        local |= v < 0 || v >= n || (k > lo && g.targets_[static_cast<std::size_t>(k) - 1] >= v);
        if (v == u) g.has_loop_[static_cast<std::size_t>(u)] = 1;
      }
    }
    if (local) bad = true;
  });
  if (bad) throw std::invalid_argument("CSR rows must be sorted, unique and in range");
  return g;
}

}  // namespace b200
}  // namespace levelrank
