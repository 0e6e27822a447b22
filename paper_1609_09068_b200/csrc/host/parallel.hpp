// Minimal fork-join helpers for the host builders (graph CSR, layout).
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstdint>
#include <thread>
#include <type_traits>
#include <vector>

#include "levelrank/graph.hpp"

namespace levelrank {
inline namespace b200 {
namespace detail {

// LR_PLAN_PROF=1: per-phase wall times of the layout build on stderr
struct PhaseClock {
  bool on = std::getenv("LR_PLAN_PROF") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[plan] %-34s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};


// Runs f(i) for i in [0, t) on t threads of the persistent host pool (the
// caller is thread 0; pool.cpp).
void pool_run_impl(int t, void (*fn)(void*, int), void* arg);
template <typename F>
void pool_run(int t, F&& f) {
  using Fn = std::remove_reference_t<F>;
  pool_run_impl(t, [](void* a, int i) { (*static_cast<Fn*>(a))(i); }, static_cast<void*>(&f));
}

// Calls f(tid, begin, end) on contiguous chunks of [0, n) from up to
// host_threads() threads (serial below `grain`).
template <typename F>
void parallel_chunks(std::int64_t n, F&& f, std::int64_t grain = 1 << 15) {
  if (n <= 0) return;
  int t = host_threads();
  if (n < grain || t <= 1) {
    f(0, std::int64_t{0}, n);
    return;
  }
  t = static_cast<int>(std::min<std::int64_t>(t, (n + grain - 1) / grain));
  pool_run(t, [&](int i) { f(i, n * i / t, n * (i + 1) / t); });
}

// A multi-hundred-MB array filled by one thread costs as much as a parallel
// pass over the edges that use it: fill (and first-touch) from all threads.
template <typename T>
void parallel_fill(T* p, std::int64_t n, T value) {
  parallel_chunks(n, [&](int, std::int64_t b, std::int64_t e) { std::fill(p + b, p + e, value); }, 1 << 18);
}
template <typename T>
uvector<T> filled(std::size_t n, T value) {
  uvector<T> v(n);
  parallel_fill(v.data(), static_cast<std::int64_t>(n), value);
  return v;
}

// Dynamic scheduling over [0, n) in blocks of `block` (for skewed work).
template <typename F>
void parallel_dynamic(std::int64_t n, std::int64_t block, F&& f) {
  if (n <= 0) return;
  const int t = host_threads();
  if (t <= 1 || n <= block) {
    for (std::int64_t i = 0; i < n; i += block) f(i, std::min(n, i + block));
    return;
  }
  std::atomic<std::int64_t> next{0};
  pool_run(t, [&](int) {
    for (;;) {
      const std::int64_t b = next.fetch_add(block);
      if (b >= n) return;
      f(b, std::min(n, b + block));
    }
  });
}

// Exclusive prefix sum in place over v[0..n); returns the total.  v has n+1
// slots when used for CSR offsets (v[n] receives the total).
template <typename T>
T exclusive_scan_inplace(T* v, std::int64_t n) {
  const int t = std::max(1, std::min<int>(host_threads(), static_cast<int>(n / (1 << 16)) + 1));
  std::vector<T> part(static_cast<std::size_t>(t) + 1, 0);
  auto run = [&](auto&& body) { pool_run(t, body); };
  run([&](int i) {
    const std::int64_t b = n * i / t, e = n * (i + 1) / t;
    T s = 0;
    for (std::int64_t k = b; k < e; ++k) s += v[k];
    part[static_cast<std::size_t>(i) + 1] = s;
  });
  for (int i = 0; i < t; ++i) part[static_cast<std::size_t>(i) + 1] += part[static_cast<std::size_t>(i)];
  run([&](int i) {
    const std::int64_t b = n * i / t, e = n * (i + 1) / t;
    T s = part[static_cast<std::size_t>(i)];
    for (std::int64_t k = b; k < e; ++k) {
      const T x = v[k];
      v[k] = s;
      s += x;
    }
  });
  return part[static_cast<std::size_t>(t)];
}

// Stable parallel LSD radix sort of items[0, n) by a 32-bit key(item),
// ascending (two 16-bit passes; the high pass is skipped when every key is
// below 2^16).
template <typename T, typename Key>
void stable_radix_sort(T* items, std::int64_t n, Key&& key) {
  if (n <= 1) return;
  if (n < (1 << 14)) {  // small inputs: a comparison sort beats the histograms
    std::stable_sort(items, items + n, [&](const T& a, const T& b) { return key(a) < key(b); });
    return;
  }
  const int t = std::max(1, std::min<int>(host_threads(), static_cast<int>(n / (1 << 15)) + 1));
  uvector<T> tmp(static_cast<std::size_t>(n));
  std::uint32_t hi_or = 0;
  for (std::int64_t i = 0; i < n && !hi_or; i += std::max<std::int64_t>(1, n / 4096)) hi_or |= key(items[i]) >> 16;
  auto run = [&](auto&& body) { pool_run(t, body); };
  if (!hi_or) {  // the sample saw no high digit: check exactly
    std::vector<std::uint32_t> any(static_cast<std::size_t>(t), 0);
    run([&](int i) {
      std::uint32_t a = 0;
      for (std::int64_t k = n * i / t; k < n * (i + 1) / t; ++k) a |= key(items[k]) >> 16;
      any[static_cast<std::size_t>(i)] = a;
    });
    for (const auto a : any) hi_or |= a;
  }
  std::vector<std::int64_t> off(static_cast<std::size_t>(t) << 16);
  T* src = items;
  T* dst = tmp.data();
  for (int pass = 0; pass < (hi_or ? 2 : 1); ++pass) {
    const int shift = 16 * pass;
    std::fill(off.begin(), off.end(), 0);
    run([&](int i) {
      std::int64_t* h = off.data() + (static_cast<std::size_t>(i) << 16);
      for (std::int64_t k = n * i / t; k < n * (i + 1) / t; ++k) ++h[(key(src[k]) >> shift) & 0xffffu];
    });
    std::int64_t acc = 0;
    for (std::size_t x = 0; x < 65536; ++x)
      for (int i = 0; i < t; ++i) {
        std::int64_t& o = off[(static_cast<std::size_t>(i) << 16) + x];
        const std::int64_t c = o;
        o = acc;
        acc += c;
      }
    run([&](int i) {
      std::int64_t* h = off.data() + (static_cast<std::size_t>(i) << 16);
      for (std::int64_t k = n * i / t; k < n * (i + 1) / t; ++k) dst[h[(key(src[k]) >> shift) & 0xffffu]++] = src[k];
    });
    std::swap(src, dst);
  }
  if (src != items) std::copy(src, src + n, items);
}

// Stable bucketed transpose into K CSRs over `nrows` rows, without atomics.
// emit(u, sink) is called for every source u in [0, n_src) -- twice, with the
// same calls both times -- and calls sink(k, row, value) for each entry of
// CSR k.  Sources are split into contiguous ascending chunks, one per thread;
// entries go to row buckets of 2^16 rows (per-thread cursors, sequential
// writes), then each bucket is counting-sorted by row.  Every row's values end
// up in emission order: source ascending, then the order emit produced them.
template <int K, typename Emit, typename PtrVec, typename ColVec>
void bucket_csr(std::int64_t n_src, std::int64_t nrows, Emit&& emit, PtrVec* ptr, ColVec* col) {
  constexpr int kShift = 16;
  const std::int64_t nb = (nrows >> kShift) + 1;
  const int t = std::max(1, std::min<int>(host_threads(), static_cast<int>(n_src / 4096) + 1));
  auto at = [&](int k, int th, std::int64_t b) {
    return (static_cast<std::size_t>(k) * static_cast<std::size_t>(t) + static_cast<std::size_t>(th)) *
               static_cast<std::size_t>(nb) + static_cast<std::size_t>(b);
  };
  std::vector<std::int64_t> cur(static_cast<std::size_t>(K) * static_cast<std::size_t>(t) * static_cast<std::size_t>(nb), 0);
  auto run = [&](auto&& body) { pool_run(t, body); };
  run([&](int th) {  // 1. per-(thread, bucket) counts
    const std::int64_t b = n_src * th / t, e = n_src * (th + 1) / t;
    for (std::int64_t u = b; u < e; ++u)
      emit(u, [&](int k, std::int64_t row, VertexId) { ++cur[at(k, th, row >> kShift)]; });
  });
  std::vector<std::int64_t> bstart(static_cast<std::size_t>(K) * static_cast<std::size_t>(nb + 1), 0);
  // a bucketed entry is its value and its row inside the bucket: 4 + 2 bytes (the
  // build is bound by memory traffic; an 8-byte (row, value) pair costs a third more)
  static_assert(kShift <= 16, "bucket-local rows are 16-bit");
  std::vector<uvector<std::uint32_t>> tmp(K);
  std::vector<uvector<std::uint16_t>> tmp_row(K);
  for (int k = 0; k < K; ++k) {  // bucket-major, then thread: stable
    std::int64_t run_total = 0;
    for (std::int64_t b = 0; b < nb; ++b) {
      bstart[static_cast<std::size_t>(k) * static_cast<std::size_t>(nb + 1) + static_cast<std::size_t>(b)] = run_total;
      for (int th = 0; th < t; ++th) {
        const std::int64_t c = cur[at(k, th, b)];
        cur[at(k, th, b)] = run_total;
        run_total += c;
      }
    }
    bstart[static_cast<std::size_t>(k) * static_cast<std::size_t>(nb + 1) + static_cast<std::size_t>(nb)] = run_total;
    tmp[static_cast<std::size_t>(k)].resize(static_cast<std::size_t>(run_total));
    tmp_row[static_cast<std::size_t>(k)].resize(static_cast<std::size_t>(run_total));
    ptr[k].resize(static_cast<std::size_t>(nrows) + 1);  // every entry written below
    col[k].resize(static_cast<std::size_t>(run_total));
  }
  run([&](int th) {  // 2. (row, value) pairs into their buckets
    const std::int64_t b = n_src * th / t, e = n_src * (th + 1) / t;
    for (std::int64_t u = b; u < e; ++u)
      emit(u, [&](int k, std::int64_t row, VertexId v) {
        const std::size_t at_ = static_cast<std::size_t>(cur[at(k, th, row >> kShift)]++);
        tmp[static_cast<std::size_t>(k)][at_] = static_cast<std::uint32_t>(v);
        tmp_row[static_cast<std::size_t>(k)][at_] = static_cast<std::uint16_t>(row & ((std::int64_t{1} << kShift) - 1));
      });
  });
  std::atomic<std::int64_t> next{0};
  run([&](int) {  // 3. counting sort of every bucket by row
    std::vector<std::int64_t> cnt(static_cast<std::size_t>(1) << kShift);
    for (;;) {
      const std::int64_t job = next.fetch_add(1);
      if (job >= K * nb) return;
      const int k = static_cast<int>(job / nb);
      const std::int64_t b = job % nb, r0 = b << kShift, r1 = std::min(nrows, (b + 1) << kShift);
      const std::int64_t s0 = bstart[static_cast<std::size_t>(k) * static_cast<std::size_t>(nb + 1) + static_cast<std::size_t>(b)];
      const std::int64_t s1 = bstart[static_cast<std::size_t>(k) * static_cast<std::size_t>(nb + 1) + static_cast<std::size_t>(b) + 1];
      if (r0 >= r1) continue;
      std::fill(cnt.begin(), cnt.begin() + (r1 - r0), 0);
      const std::uint32_t* src = tmp[static_cast<std::size_t>(k)].data();
      const std::uint16_t* srow = tmp_row[static_cast<std::size_t>(k)].data();
      for (std::int64_t i = s0; i < s1; ++i) ++cnt[srow[i]];
      std::int64_t pos = s0;
      for (std::int64_t r = r0; r < r1; ++r) {
        ptr[k][static_cast<std::size_t>(r)] = pos;
        const std::int64_t c = cnt[static_cast<std::size_t>(r - r0)];
        cnt[static_cast<std::size_t>(r - r0)] = pos;
        pos += c;
      }
      VertexId* out = col[k].data();
      for (std::int64_t i = s0; i < s1; ++i) out[cnt[srow[i]]++] = static_cast<VertexId>(src[i]);
    }
  });
  for (int k = 0; k < K; ++k)
    ptr[k][static_cast<std::size_t>(nrows)] = bstart[static_cast<std::size_t>(k) * static_cast<std::size_t>(nb + 1) + static_cast<std::size_t>(nb)];
}

}  // namespace detail
}  // namespace b200
}  // namespace levelrank
