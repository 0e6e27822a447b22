// solve_large_scc with PowerSeriesStats (proj/src/solvers.cpp:128-162,
// proj/include/levelrank/solvers.hpp:23-27): the instrumented form of the
// power series for the unit-solver API, when a caller asks for the L1 norm of
// every increment and the smallest increment entry.  One thread per row pulls
// its in-edges in source order (the order solve_large_scc's scatter over
// unit.edges adds them, so rows are bit-exact), each CTA reduces its rows'
// sum / min / max, and one CTA folds the CTA partials in a fixed order.  The
// host drives the iterations (one 24-byte read-back each): this path exists
// for the statistics; the solves themselves go through the level loop.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "lr_cuda.h"

namespace lrerr {
void set(const std::string& msg);
}

namespace {

constexpr int kRows = 256;

__global__ void k_series_step(int m, const long long* __restrict__ ptr, const int* __restrict__ src,
                              const double* __restrict__ pf, const double* __restrict__ inc, double* next,
                              double* rank, double* part) {
  __shared__ double s_sum[kRows], s_min[kRows], s_max[kRows];
  const int i = blockIdx.x * kRows + threadIdx.x;
  double y = 0.0;
  if (i < m) {
    for (long long e = ptr[i]; e < ptr[i + 1]; ++e) {
      const int a = src[e];
      y += pf[a] * inc[a];
    }
    next[i] = y;
    rank[i] += y;
  }
  s_sum[threadIdx.x] = i < m ? fabs(y) : 0.0;
  s_min[threadIdx.x] = i < m ? y : INFINITY;
  s_max[threadIdx.x] = i < m ? fabs(y) : 0.0;
  __syncthreads();
  for (int w = kRows / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s_sum[threadIdx.x] += s_sum[threadIdx.x + w];
      s_min[threadIdx.x] = fmin(s_min[threadIdx.x], s_min[threadIdx.x + w]);
      s_max[threadIdx.x] = fmax(s_max[threadIdx.x], s_max[threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = s_sum[0];
    part[3 * blockIdx.x + 1] = s_min[0];
    part[3 * blockIdx.x + 2] = s_max[0];
  }
}

__global__ void k_series_fold(int nb, const double* part, double* out3) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0, mn = INFINITY, mx = 0.0;
  for (int b = 0; b < nb; ++b) {
    s += part[3 * b];
    mn = fmin(mn, part[3 * b + 1]);
    mx = fmax(mx, part[3 * b + 2]);
  }
  out3[0] = s;
  out3[1] = mn;
  out3[2] = mx;
}

struct Buf {
  void* p = nullptr;
  ~Buf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, n ? n : 1); }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

#define LR_SER_TRY(expr)                                                       \
  do {                                                                         \
    const cudaError_t e_ = (expr);                                             \
    if (e_ != cudaSuccess) {                                                   \
      lrerr::set(std::string("CUDA: ") + cudaGetErrorString(e_) + " (" #expr ")"); \
      return LR_ECUDA;                                                         \
    }                                                                          \
  } while (0)

}  // namespace

// Pull CSR of the unit (row i's in-edge sources ascending), push factors,
// start weights.  Fills ranks[m], *iterations, l1[min(iterations, cap)] and
// *min_entry; LR_ENOCONV past the iteration cap (solvers.cpp:159).
extern "C" lr_status lr_series_stats_csr(int device, int32_t m, const long long* ptr, const int32_t* src,
                                         const double* pf, const double* w, double tol, int64_t cap,
                                         double* ranks, int64_t* iterations, double* l1, int64_t l1_cap,
                                         double* min_entry) {
  *iterations = 0;
  *min_entry = std::numeric_limits<double>::infinity();
  if (m <= 0) return LR_OK;
  LR_SER_TRY(cudaSetDevice(device));
  const long long nnz = ptr[m];
  const int nb = (m + kRows - 1) / kRows;
  Buf d_ptr, d_src, d_pf, d_a, d_b, d_rank, d_part, d_out;
  LR_SER_TRY(d_ptr.alloc(sizeof(long long) * (static_cast<size_t>(m) + 1)));
  LR_SER_TRY(d_src.alloc(sizeof(int) * static_cast<size_t>(nnz)));
  LR_SER_TRY(d_pf.alloc(sizeof(double) * static_cast<size_t>(m)));
  LR_SER_TRY(d_a.alloc(sizeof(double) * static_cast<size_t>(m)));
  LR_SER_TRY(d_b.alloc(sizeof(double) * static_cast<size_t>(m)));
  LR_SER_TRY(d_rank.alloc(sizeof(double) * static_cast<size_t>(m)));
  LR_SER_TRY(d_part.alloc(sizeof(double) * 3 * static_cast<size_t>(nb)));
  LR_SER_TRY(d_out.alloc(sizeof(double) * 3));
  LR_SER_TRY(cudaMemcpy(d_ptr.p, ptr, sizeof(long long) * (static_cast<size_t>(m) + 1), cudaMemcpyHostToDevice));
  if (nnz) LR_SER_TRY(cudaMemcpy(d_src.p, src, sizeof(int) * static_cast<size_t>(nnz), cudaMemcpyHostToDevice));
  LR_SER_TRY(cudaMemcpy(d_pf.p, pf, sizeof(double) * static_cast<size_t>(m), cudaMemcpyHostToDevice));
  LR_SER_TRY(cudaMemcpy(d_a.p, w, sizeof(double) * static_cast<size_t>(m), cudaMemcpyHostToDevice));
  LR_SER_TRY(cudaMemcpy(d_rank.p, w, sizeof(double) * static_cast<size_t>(m), cudaMemcpyHostToDevice));
  double* inc = d_a.as<double>();
  double* nxt = d_b.as<double>();
  double out[3];
  for (;;) {  // do { ... } while (max|inc| >= tol)  (solvers.cpp:146-160)
    k_series_step<<<nb, kRows>>>(m, d_ptr.as<long long>(), d_src.as<int>(), d_pf.as<double>(), inc, nxt,
                                 d_rank.as<double>(), d_part.as<double>());
    k_series_fold<<<1, 32>>>(nb, d_part.as<double>(), d_out.as<double>());
    LR_SER_TRY(cudaGetLastError());
    LR_SER_TRY(cudaMemcpy(out, d_out.p, sizeof out, cudaMemcpyDeviceToHost));
    std::swap(inc, nxt);
    const int64_t it = ++*iterations;
    if (it <= l1_cap && l1) l1[it - 1] = out[0];
    *min_entry = std::fmin(*min_entry, out[1]);
    if (it > cap) {
      lrerr::set("power series failed to converge");
      return LR_ENOCONV;
    }
    if (!(out[2] >= tol)) break;
  }
  LR_SER_TRY(cudaMemcpy(ranks, d_rank.p, sizeof(double) * static_cast<size_t>(m), cudaMemcpyDeviceToHost));
  return LR_OK;
}
