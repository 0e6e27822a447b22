// sm_100a kernels of the level-scheduled PageRank solve.  Everything here is
// fp64 and HBM/latency bound; no tensor cores (nothing on the path is a dense
// contraction).  Accumulation orders are chosen so that every term and every
// summation order matches the reference's CPU loops wherever a row is summed
// by one thread; the file is compiled with
// --fmad=false so no multiply-add is contracted behind our back.
#include <cuda_runtime.h>

#include <cstdint>

#include "devutil.cuh"
#include "kernels.cuh"

namespace lrk {
namespace {

__device__ __forceinline__ unsigned long long dbits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}
__device__ __forceinline__ double bitsd(unsigned long long b) {
  return __longlong_as_double(static_cast<long long>(b));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide max; `red` holds blockDim/32 doubles.  All threads get the result.
__device__ __forceinline__ double block_max(double v, double* red) {
  v = warp_max(v);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) red[warp] = v;
  __syncthreads();
  double m = red[0];
  for (int i = 1; i < nw; ++i) m = fmax(m, red[i]);
  return m;
}
// Block-wide sum in a fixed order (deterministic).
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) red[warp] = v;
  __syncthreads();
  double s = red[0];
  for (int i = 1; i < nw; ++i) s += red[i];
  return s;
}

// ----------------------------------------------------------------- prep
// Weight checks of engine.cpp:94-97,112 (negative -> error bit, max == 0 ->
// all_weights_zero) and the per-row push factor c / walk_out_degree
// (solvers.cpp:136-138; 0 for dangling rows, which never push).
__global__ void k_prep(DeviceLayout L, const double* __restrict__ w, const SolveParams* __restrict__ p,
                       double* __restrict__ pf, DevStatus* st) {
  __shared__ double red[32];
  const double c = p->c;
  double wmax = 0.0;
  bool neg = false;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L.n; i += gridDim.x * blockDim.x) {
    const double x = w[i];
    neg |= x < 0.0;
    wmax = fmax(wmax, x);
    const int d = L.deg[i];
    pf[i] = d > 0 ? c / static_cast<double>(d) : 0.0;
  }
  if (__syncthreads_or(neg) && threadIdx.x == 0) atomicOr(&st->err, kErrNegW);
  const double m = block_max(wmax, red);
  if (threadIdx.x == 0 && m > 0.0) atomicMax(&st->wmax_bits, dbits(m));
}

__device__ __forceinline__ void cross_finish(const DeviceLayout& L, int row, double acc, double c,
                                             const double* __restrict__ pf, double* rank, double* s0) {
  const std::uint8_t k = L.rowkind[row];
  if (k == kSingle && L.loop[row]) acc /= 1.0 - c / static_cast<double>(L.deg[row]);
  rank[row] = acc;
  if (k == kLargeGrid) s0[row] = pf[row] * acc;
}

// Pull rows with more than kCrossLight in-edges: one warp per kCrossSeg-edge
// slice (every gather of a slice in flight together); slices of one row
// combine in slice order in the last one to finish.
// kCac = false: cross in-edges of K1 (base = w, finish = cross_finish);
// kCac = true : intra in-edges of a large-CAC depth slice (base = rank).
// Same terms as the one-thread paths, tree-summed.
template <bool kCac>
__global__ void k_pull_heavy(DeviceLayout L, const CrossTask* __restrict__ tasks, int ntasks,
                             const double* __restrict__ w, const SolveParams* __restrict__ p,
                             const double* __restrict__ pf, double* rank, double* __restrict__ s0, double* parts,
                             int* cnts) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= ntasks) return;
  const CrossTask x = tasks[t];
  const double c = p->c;
  const int* src = kCac ? L.isrc : L.xsrc;
  // kCrossSeg = 8 x 32 edges: indices, then all gathers, then the terms
  constexpr int kPer = kCrossSeg / 32;
  int s[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) s[k] = lane + 32 * k < x.cnt ? __ldg(src + x.e_begin + lane + 32 * k) : -1;
  double rv[kPer];
  int dv[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    rv[k] = s[k] >= 0 ? rank[s[k]] : 0.0;
    dv[k] = s[k] >= 0 ? __ldg(L.deg + s[k]) : 1;
  }
  double sum = 0.0;
#pragma unroll
  for (int k = 0; k < kPer; ++k)
    if (s[k] >= 0) sum += c * rv[k] / static_cast<double>(dv[k]);
  sum = dev::warp_sum(sum);
  if (lane != 0) return;
  double y = sum;
  if (x.nseg > 1) {
    parts[x.part_begin + x.seg] = sum;
    __threadfence();
    if (atomicAdd(cnts + x.slot, 1) != x.nseg - 1) return;
    __threadfence();
    y = 0.0;
    for (int k = 0; k < x.nseg; ++k) y += __ldcg(parts + x.part_begin + k);
    cnts[x.slot] = 0;
  }
  if (kCac) {
    double acc = rank[x.row] + y;
    if (L.loop[x.row]) acc /= 1.0 - c / static_cast<double>(L.deg[x.row]);
    rank[x.row] = acc;
  } else {
    cross_finish(L, x.row, w[L.vertex_of[x.row]] + y, c, pf, rank, s0);
  }
}

// ------------------------------------------------------------------ CAC
// One depth slice of a large CAC across the whole grid (the slice's parents
// are final: earlier slices ran in earlier launches).
__global__ void k_cac_slice(DeviceLayout L, int row_begin, int row_end, const SolveParams* __restrict__ p,
                            double* rank) {
  const int r = row_begin + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= row_end) return;
  const long long e1 = L.iptr[r + 1];
  if (e1 - L.iptr[r] > kCrossLight) return;  // heavy rows: k_pull_heavy<true>
  const double c = p->c;
  double acc = rank[r];
  for (long long e = L.iptr[r]; e < e1; ++e) {
    const int s = __ldg(L.isrc + e);
    acc += rank[s] * c / static_cast<double>(__ldg(L.deg + s));
  }
  if (L.loop[r]) acc /= 1.0 - c / static_cast<double>(L.deg[r]);
  rank[r] = acc;
}

// ------------------------------------------------------------ small SCC
// K5: exact dense solve of (I - cA^T) r = w per SccSmall unit
// (solve_dense_system, solvers.cpp:92-108).  The matrix is strictly
// diagonally dominant by columns (column a holds 1 on the diagonal and at most
// c < 1 of off-diagonal mass), so partial pivoting never swaps rows and the
// reference's partialPivLu reduces to plain Gaussian elimination, done here in
// shared memory.  Residual check of solvers.cpp:103-106 -> kErrDegen.
__global__ void k_small(DeviceLayout L, const SccTask* __restrict__ tasks, int ntasks, int ld,
                        const double* __restrict__ pf, double* rank, double* scratch, DevStatus* st) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  double* M = scratch ? scratch + static_cast<size_t>(blockIdx.x) * ld * (ld + 2) : sm;
  double* rhs = M + static_cast<size_t>(ld) * ld;
  double* fcol = rhs + ld;
  const int tid = threadIdx.x, bs = blockDim.x;
  for (int task = blockIdx.x; task < ntasks; task += gridDim.x) {
    const SccTask t = tasks[task];
    const int rb = t.row_begin, m = t.row_end - t.row_begin;
    __syncthreads();
    for (int i = tid; i < m * ld; i += bs) M[i] = 0.0;
    __syncthreads();
    for (int b = tid; b < m; b += bs) {
      M[b * ld + b] = 1.0;
      rhs[b] = rank[rb + b];
    }
    __syncthreads();
    for (int b = tid; b < m; b += bs) {
      const long long e1 = L.iptr[rb + b + 1];
      for (long long e = L.iptr[rb + b]; e < e1; ++e) {
        const int s = L.isrc[e];
        M[b * ld + (s - rb)] -= pf[s];
      }
    }
    for (int k = 0; k < m; ++k) {
      __syncthreads();
      const double piv = M[k * ld + k];
      for (int i = k + 1 + tid; i < m; i += bs) {
        const double f = M[i * ld + k] / piv;
        fcol[i] = f;
        rhs[i] -= f * rhs[k];
      }
      __syncthreads();
      const int w = m - k - 1;
      for (int idx = tid; idx < w * w; idx += bs) {
        const int i = k + 1 + idx / w, j = k + 1 + idx % w;
        M[i * ld + j] -= fcol[i] * M[k * ld + j];
      }
    }
    for (int i = m - 1; i >= 0; --i) {
      __syncthreads();
      const double xi = rhs[i] / M[i * ld + i];
      __syncthreads();
      if (tid == 0) rhs[i] = xi;
      for (int r = tid; r < i; r += bs) rhs[r] -= M[r * ld + i] * xi;
    }
    __syncthreads();
    double res = 0.0, wm = 0.0, xm = 0.0;
    for (int b = tid; b < m; b += bs) {
      const double wb = rank[rb + b];
      double acc = rhs[b];
      const long long e1 = L.iptr[rb + b + 1];
      for (long long e = L.iptr[rb + b]; e < e1; ++e) {
        const int s = L.isrc[e];
        acc -= pf[s] * rhs[s - rb];
      }
      res = fmax(res, fabs(acc - wb));
      wm = fmax(wm, fabs(wb));
      xm = fmax(xm, fabs(rhs[b]));
    }
    res = block_max(res, red);
    __syncthreads();
    wm = block_max(wm, red);
    __syncthreads();
    xm = block_max(xm, red);
    if (tid == 0 && !(res <= 1e-8 * (1.0 + wm + xm))) atomicOr(&st->err, kErrDegen);
    for (int b = tid; b < m; b += bs) rank[rb + b] = rhs[b];
  }
}

// --------------------------------------------------------------- output
// R3 back to vertex order and fixed-order partial sums for the R1 total.
__global__ void k_output(DeviceLayout L, const double* __restrict__ rank, double* __restrict__ r3,
                         double* __restrict__ partial) {
  __shared__ double red[kOutBlock / 32];
  const int v = blockIdx.x * kOutBlock + threadIdx.x;
  double x = 0.0;
  if (v < L.n) {
    x = rank[L.row_of[v]];
    r3[v] = x;
  }
  const double s = block_sum(x, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void k_sum_partials(const double* __restrict__ partial, int nparts, double* total) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partial[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *total = s;
}

// R1 = R3 / ||R3||_1 (r3 >= 0); zero when the total is zero.
__global__ void k_scale(const double* __restrict__ r3, double* __restrict__ r1, int n, const double* total) {
  const double t = *total;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    r1[v] = t > 0.0 ? r3[v] / t : 0.0;
}

// propagate_weights (engine.cpp:83-87) for the standalone API: one thread per
// destination, its edges in input order.
__global__ void k_propagate(const int* __restrict__ order, const long long* __restrict__ seg_ptr, int nseg,
                            const int* __restrict__ src, const int* __restrict__ dst, const int* __restrict__ deg,
                            const double* __restrict__ ranks, double c, double* weights) {
  const int sgi = blockIdx.x * blockDim.x + threadIdx.x;
  if (sgi >= nseg) return;
  const long long e0 = seg_ptr[sgi], e1 = seg_ptr[sgi + 1];
  const int d = dst[order[e0]];
  double acc = weights[d];
  for (long long e = e0; e < e1; ++e) {
    const int k = order[e];
    acc += c * ranks[src[k]] / static_cast<double>(deg[k]);
  }
  weights[d] = acc;
}

int blocks_for(long long n, int threads) { return static_cast<int>((n + threads - 1) / threads); }

}  // namespace

void launch_prep(const DeviceLayout& L, const double* w, const SolveParams* p, double* pf, DevStatus* st,
                 cudaStream_t s) {
  if (L.n == 0) return;
  const int grid = blocks_for(L.n, 256) < 148 * 8 ? blocks_for(L.n, 256) : 148 * 8;
  k_prep<<<grid, 256, 0, s>>>(L, w, p, pf, st);
}

void launch_cross_heavy(const DeviceLayout& L, const CrossTask* tasks, int ntasks, const double* w,
                        const SolveParams* p, const double* pf, double* rank, double* s0, double* parts, int* cnts,
                        cudaStream_t s) {
  if (ntasks == 0) return;
  k_pull_heavy<false><<<blocks_for(ntasks, 8), 256, 0, s>>>(L, tasks, ntasks, w, p, pf, rank, s0, parts, cnts);
}

void launch_cac_heavy(const DeviceLayout& L, const CrossTask* tasks, int ntasks, const SolveParams* p, double* rank,
                      double* parts, int* cnts, cudaStream_t s) {
  if (ntasks == 0) return;
  k_pull_heavy<true><<<blocks_for(ntasks, 8), 256, 0, s>>>(L, tasks, ntasks, nullptr, p, nullptr, rank, nullptr,
                                                           parts, cnts);
}

void launch_cac_slice(const DeviceLayout& L, int row_begin, int row_end, const SolveParams* p, double* rank,
                      cudaStream_t s) {
  if (row_end <= row_begin) return;
  k_cac_slice<<<blocks_for(row_end - row_begin, 256), 256, 0, s>>>(L, row_begin, row_end, p, rank);
}

void launch_small(const DeviceLayout& L, const SccTask* tasks, int ntasks, int max_m, const double* pf,
                  double* rank, double* scratch, DevStatus* st, cudaStream_t s) {
  if (ntasks == 0) return;
  const int ld = max_m + 1;
  const size_t bytes = static_cast<size_t>(ld) * (ld + 2) * sizeof(double);
  if (scratch == nullptr) {
    k_small<<<ntasks, 256, bytes, s>>>(L, tasks, ntasks, ld, pf, rank, nullptr, st);
  } else {
    const int grid = ntasks < kSmallScratchBlocks ? ntasks : kSmallScratchBlocks;
    k_small<<<grid, 256, 0, s>>>(L, tasks, ntasks, ld, pf, rank, scratch, st);
  }
}

template <typename K>
static cudaError_t allow_dynamic_smem(K kernel, int optin) {
  cudaFuncAttributes a{};
  cudaError_t e = cudaFuncGetAttributes(&a, kernel);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin - static_cast<int>(a.sharedSizeBytes));
}

cudaError_t configure_kernels() {
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  return allow_dynamic_smem(k_small, optin);
}

void launch_output(const DeviceLayout& L, const double* rank, double* r3, double* partial, int nparts,
                   cudaStream_t s) {
  if (nparts == 0) return;
  k_output<<<nparts, kOutBlock, 0, s>>>(L, rank, r3, partial);
}

void launch_normalize(const double* r3, double* r1, int n, const double* partial, int nparts, double* total,
                      cudaStream_t s) {
  k_sum_partials<<<1, 1024, 0, s>>>(partial, nparts, total);
  if (r1 && n > 0) k_scale<<<blocks_for(n, 256) < 148 * 16 ? blocks_for(n, 256) : 148 * 16, 256, 0, s>>>(r3, r1, n, total);
}

void launch_propagate(const int* order, const long long* seg_ptr, int nseg, const int* src, const int* dst,
                      const int* deg, const double* ranks, double c, double* weights, cudaStream_t s) {
  if (nseg == 0) return;
  k_propagate<<<blocks_for(nseg, 256), 256, 0, s>>>(order, seg_ptr, nseg, src, dst, deg, ranks, c, weights);
}

}  // namespace lrk
