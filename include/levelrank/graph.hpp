// levelrank-b200 host API: graph core.
//
// Drop-in for the reference's proj/include/levelrank/graph.hpp:1-107 (same
// names, argument meaning and exceptions), re-implemented for large inputs:
// from_edges runs a multi-threaded count/scatter/sort-rows build instead of one
// global std::sort.  Lives in levelrank::b200 (an inline namespace), so code
// written against `levelrank::Graph` recompiles unchanged while the symbols
// never collide with a reference build loaded in the same process.
#pragma once

#include <sys/mman.h>

#include <cstdlib>
#include <new>
#include <cstdint>
#include <iosfwd>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace levelrank {
inline namespace b200 {

using VertexId = std::int32_t;
using EdgeId = std::int64_t;

/// std::vector whose resize() leaves new elements default-initialised (no
/// zero fill): the host builders size multi-GB arrays and then write every
/// element from many threads, which also spreads the first-touch page faults.
template <typename T>
struct UninitAllocator : std::allocator<T> {
  using value_type = T;
  UninitAllocator() = default;
  template <typename U>
  UninitAllocator(const UninitAllocator<U>&) noexcept {}
  template <typename U>
  struct rebind {
    using other = UninitAllocator<U>;
  };
  template <typename U, typename... Args>
  void construct(U* p, Args&&... args) {
    if constexpr (sizeof...(Args) == 0) ::new (static_cast<void*>(p)) U;
    else ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
  // Large arrays (per-vertex and per-edge tables that the plan build reads at
  // random) ask for transparent huge pages: with 4 KB pages a random read of a
  // 268 MB table misses the TLB nearly every time.
  static constexpr std::size_t kHugeBytes = std::size_t{1} << 22, kHugeAlign = std::size_t{1} << 21;
  T* allocate(std::size_t n) {
    const std::size_t bytes = n * sizeof(T);
    if (bytes < kHugeBytes) return std::allocator<T>::allocate(n);
    void* p = nullptr;
    if (n > static_cast<std::size_t>(-1) / sizeof(T) || posix_memalign(&p, kHugeAlign, bytes) != 0) throw std::bad_alloc();
    madvise(p, bytes, MADV_HUGEPAGE);
    return static_cast<T*>(p);
  }
  void deallocate(T* p, std::size_t n) noexcept {
    if (n * sizeof(T) < kHugeBytes) std::allocator<T>::deallocate(p, n);
    else std::free(p);
  }
};
template <typename T>
using uvector = std::vector<T, UninitAllocator<T>>;

/// graph.hpp:19 -- n = max id + 1 must fit in VertexId.
inline constexpr VertexId kMaxVertexId = 2147483646;

/// graph.hpp:23 -- Ignore drops self-loops from the walk; Keep walks them.
enum class LoopPolicy { Ignore, Keep };

class ParseError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class IoError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

/// Compressed out-adjacency, rows sorted and duplicate-free (graph.hpp:39-76).
class Graph {
 public:
  Graph() = default;

  /// graph.cpp:14-36 semantics: range check (std::invalid_argument), dedup,
  /// sorted rows, loop flags.  Multi-threaded.
  static Graph from_edges(VertexId n, std::vector<std::pair<VertexId, VertexId>> edges,
                          LoopPolicy policy = LoopPolicy::Ignore);
  /// Same, from two parallel arrays (no pair vector materialised).
  static Graph from_edge_arrays(VertexId n, const VertexId* src, const VertexId* dst, EdgeId m,
                                LoopPolicy policy = LoopPolicy::Ignore);
  /// Adopts an existing CSR; rows must be sorted and duplicate-free
  /// (checked, std::invalid_argument otherwise).
  static Graph from_csr(VertexId n, std::vector<EdgeId> offsets, std::vector<VertexId> targets,
                        LoopPolicy policy = LoopPolicy::Ignore);

  [[nodiscard]] VertexId vertex_count() const noexcept { return n_; }
  [[nodiscard]] EdgeId edge_count() const noexcept { return static_cast<EdgeId>(targets_.size()); }
  [[nodiscard]] LoopPolicy loop_policy() const noexcept { return policy_; }

  [[nodiscard]] std::span<const VertexId> out_neighbors(VertexId u) const {
    return {targets_.data() + offsets_[u], targets_.data() + offsets_[u + 1]};
  }
  [[nodiscard]] VertexId out_degree(VertexId u) const {
    return static_cast<VertexId>(offsets_[u + 1] - offsets_[u]);
  }
  [[nodiscard]] bool has_loop(VertexId u) const { return has_loop_[u] != 0; }
  /// graph.hpp:61-65.
  [[nodiscard]] VertexId walk_out_degree(VertexId u) const {
    VertexId d = out_degree(u);
    if (policy_ == LoopPolicy::Ignore && has_loop(u)) --d;
    return d;
  }

  [[nodiscard]] const EdgeId* offsets_data() const noexcept { return offsets_.data(); }
  [[nodiscard]] const VertexId* targets_data() const noexcept { return targets_.data(); }
  [[nodiscard]] const std::uint8_t* loop_data() const noexcept { return has_loop_.data(); }

 private:
  VertexId n_ = 0;
  std::vector<EdgeId> offsets_ = {0};
  std::vector<VertexId> targets_;
  std::vector<std::uint8_t> has_loop_;
  LoopPolicy policy_ = LoopPolicy::Ignore;
};

/// graph.cpp:54-99: "src<TAB>dst" lines, '#' comments, LF/CRLF; dense ids or
/// compaction in sorted order.  ParseError on malformed or empty input.
Graph parse_edge_list(std::istream& in, bool dense_ids, LoopPolicy policy = LoopPolicy::Ignore);
/// The same format from a byte buffer (the reader behind both entry points:
/// chunked over the host threads, errors name the first bad line).
Graph parse_edge_buffer(const char* data, std::size_t len, bool dense_ids,
                        LoopPolicy policy = LoopPolicy::Ignore);
/// graph.cpp:101-105 (the file is mmap'ed); IoError if it cannot be opened.
Graph load_edge_list(const std::string& path, bool dense_ids, LoopPolicy policy = LoopPolicy::Ignore);

/// Worker threads used by the host builders (LR_THREADS env var, else
/// hardware concurrency).
int host_threads();

}  // namespace b200
}  // namespace levelrank
