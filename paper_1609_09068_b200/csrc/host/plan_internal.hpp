// Plan-build internals shared by the partition and the layout: the graph's
// in-edge lists are built once (by the partition, which needs them for its
// backward reachability and wavefront release) and reused by the layout for
// its per-row pull lists, instead of a second transpose of every edge.
#pragma once

#include <cstdint>
#include <vector>

#include "levelrank/partition.hpp"
#include "levelrank/schedule.hpp"

namespace levelrank {
inline namespace b200 {
namespace detail {

struct InEdges {
  uvector<EdgeId> off;    // n + 1
  uvector<VertexId> src;  // per target vertex: sources ascending, self-loops left out
  // One bit per out-edge (graph order) and per in-edge (order of `src`): set
  // when the edge leaves its SCC.  A clear bit means both ends lie in one SCC,
  // hence in one final component (absorption only merges single-vertex
  // components), so the layout looks components up only for the set bits --
  // 1.5 % of the edges of a scale-free graph with a giant SCC.  Empty when the
  // partition did not record them.
  uvector<std::uint64_t> cross_out, cross_in;
};

// bit writer for one thread's edge range: words are shared at range boundaries,
// so set bits are flushed with an atomic OR, one per touched word
class CrossBits {
 public:
  explicit CrossBits(std::uint64_t* words) : w_(words) {}
  ~CrossBits() { flush(); }
  void set(EdgeId k) {
    const EdgeId wi = k >> 6;
    if (wi != cur_) {
      flush();
      cur_ = wi;
    }
    acc_ |= std::uint64_t{1} << (k & 63);
  }
  void flush() {
    if (acc_) __atomic_fetch_or(&w_[cur_], acc_, __ATOMIC_RELAXED);
    acc_ = 0;
  }

 private:
  std::uint64_t* w_;
  EdgeId cur_ = -1;
  std::uint64_t acc_ = 0;
};

// calls f(k) for every set bit k of [k0, k1)
template <typename F>
inline void for_cross_bits(const std::uint64_t* words, EdgeId k0, EdgeId k1, F&& f) {
  if (k0 >= k1) return;
  for (EdgeId wi = k0 >> 6; wi <= (k1 - 1) >> 6; ++wi) {
    std::uint64_t x = words[wi];
    if (wi == (k0 >> 6)) x &= ~std::uint64_t{0} << (k0 & 63);
    if (wi == ((k1 - 1) >> 6) && ((k1 & 63) != 0)) x &= (std::uint64_t{1} << (k1 & 63)) - 1;
    for (; x; x &= x - 1) f((wi << 6) + __builtin_ctzll(x));
  }
}
inline EdgeId count_cross_bits(const std::uint64_t* words, EdgeId k0, EdgeId k1) {
  EdgeId n = 0;
  if (k0 >= k1) return 0;
  for (EdgeId wi = k0 >> 6; wi <= (k1 - 1) >> 6; ++wi) {
    std::uint64_t x = words[wi];
    if (wi == (k0 >> 6)) x &= ~std::uint64_t{0} << (k0 & 63);
    if (wi == ((k1 - 1) >> 6) && ((k1 & 63) != 0)) x &= (std::uint64_t{1} << (k1 & 63)) - 1;
    n += __builtin_popcountll(x);
  }
  return n;
}

Partition find_components_with_in_edges(const Graph& g, PartitionStats* stats, InEdges& in);
Layout build_layout_from(const Graph& g, const Partition& p, VertexId small_threshold, const InEdges& in);

}  // namespace detail
}  // namespace b200
}  // namespace levelrank
