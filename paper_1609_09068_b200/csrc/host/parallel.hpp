// Minimal fork-join helpers for the host builders (graph CSR, layout).
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <thread>
#include <vector>

#include "levelrank/graph.hpp"

namespace levelrank {
inline namespace b200 {
namespace detail {

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
  std::vector<std::thread> pool;
  pool.reserve(static_cast<std::size_t>(t));
  for (int i = 0; i < t; ++i) {
    const std::int64_t b = n * i / t, e = n * (i + 1) / t;
    pool.emplace_back([&f, i, b, e] { f(i, b, e); });
  }
  for (auto& th : pool) th.join();
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
  std::vector<std::thread> pool;
  for (int i = 0; i < t; ++i)
    pool.emplace_back([&] {
      for (;;) {
        const std::int64_t b = next.fetch_add(block);
        if (b >= n) return;
        f(b, std::min(n, b + block));
      }
    });
  for (auto& th : pool) th.join();
}

// Exclusive prefix sum in place over v[0..n); returns the total.  v has n+1
// slots when used for CSR offsets (v[n] receives the total).
template <typename T>
T exclusive_scan_inplace(T* v, std::int64_t n) {
  const int t = std::max(1, std::min<int>(host_threads(), static_cast<int>(n / (1 << 16)) + 1));
  std::vector<T> part(static_cast<std::size_t>(t) + 1, 0);
  std::vector<std::thread> pool;
  auto run = [&](auto&& body) {
    pool.clear();
    for (int i = 0; i < t; ++i) pool.emplace_back(body, i);
    for (auto& th : pool) th.join();
  };
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

}  // namespace detail
}  // namespace b200
}  // namespace levelrank
