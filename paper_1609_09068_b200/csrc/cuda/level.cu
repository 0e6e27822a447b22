// The fused per-level kernel: one launch solves every unit of a level that
// fits a CTA.  Deep DAGs (config 4: 1000 levels of
// ~16k vertices, a few hundred small components each) are bound by per-level
// latency, not bandwidth, so everything a level needs -- the cross-level
// gather of its start weights (K1), singleton rows, CACs (K3), small SCCs
// (K5) and CTA-sized large SCCs (K4a) -- runs as heterogeneous CTAs of a
// single launch.  Each unit task gathers its own rows' cross in-edges first,
// so no grid-wide barrier is needed between K1 and the unit solves.
//
// Accumulation orders are the reference's wherever one thread sums a row
// (cross in-edges in propagate_weights order, CAC parents in Kahn order, SCC
// in-edges in source order); rows with more than kCrossLight in-edges are
// summed by a warp butterfly, and rows with more than kCrossSplit cross
// in-edges by the separate segment kernel (k_pull_heavy) launched before.
#include <cuda_runtime.h>

#include <climits>

#include <cstdint>
#include <cstdio>

#include <type_traits>

#include "devutil.cuh"
#include "kernels.cuh"

namespace lrk {
namespace {

using namespace dev;

constexpr int kThreads = 256;
constexpr int kWarpsPer = kThreads / 32;

// ------------------------------------------------------------- K1 pieces
// w + sum over cross in-edges of (c * r_src) / deg_src, reference order.
__device__ __forceinline__ double cross_serial(const DeviceLayout& L, int row, const double* __restrict__ w, double c,
                                               const double* rank, long long e0, long long e1) {
  double acc = w[L.vertex_of[row]];
#pragma unroll 4
  for (long long e = e0; e < e1; ++e) {
    const int s = __ldg(L.xsrc + e);
    acc += c * rank[s] / static_cast<double>(__ldg(L.deg + s));
  }
  return acc;
}

__device__ __forceinline__ double cross_warp_sum(const DeviceLayout& L, const double* rank, double c, long long e0,
                                                 long long e1, int lane) {
  double y = 0.0;
  for (long long e = e0 + lane; e < e1; e += 32) {
    const int s = __ldg(L.xsrc + e);
    y += c * rank[s] / static_cast<double>(__ldg(L.deg + s));
  }
  return warp_sum(y);
}

// start weight finishes: singletons are solved (solvers.cpp:23-35), grid
// SccLarge rows get their first pushed value s0 = pf * w
__device__ __forceinline__ void row_finish(const DeviceLayout& L, int row, double acc, double c,
                                           const double* __restrict__ pf, double* rank, double* s0) {
  const std::uint8_t k = L.rowkind[row];
  if (k == kSingle && L.loop[row]) acc /= 1.0 - c / static_cast<double>(L.deg[row]);
  rank[row] = acc;
  if (k == kLargeGrid) s0[row] = pf[row] * acc;
}

// Start weights of rows [r0, r1) by `width` threads at offset `tid` (a whole
// CTA or one warp; warp-level cooperation for heavy rows happens inside each
// warp of the group).  Rows above kCrossSplit were done by k_pull_heavy.
__device__ void cross_rows(const DeviceLayout& L, int r0, int r1, const double* __restrict__ w, double c,
                           const double* __restrict__ pf, double* rank, double* s0, int tid, int width) {
  for (int r = r0 + tid; r < r1; r += width) {
    const long long e0 = L.xptr[r], e1 = L.xptr[r + 1];
    if (e1 - e0 > kCrossLight) continue;
    row_finish(L, r, cross_serial(L, r, w, c, rank, e0, e1), c, pf, rank, s0);
  }
  // heavy rows: one warp each
  const int lane = threadIdx.x & 31;
  const int wid = tid >> 5, nw = width >> 5;
  for (int base = r0 + wid * 32; base < r1; base += nw * 32) {
    const int r = base + lane;
    long long d = 0;
    if (r < r1) d = L.xptr[r + 1] - L.xptr[r];
    unsigned mask = __ballot_sync(0xffffffffu, d > kCrossLight && d <= kCrossSplit);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const int row = base + src;
      const double y = cross_warp_sum(L, rank, c, L.xptr[row], L.xptr[row + 1], lane);
      if (lane == 0) row_finish(L, row, w[L.vertex_of[row]] + y, c, pf, rank, s0);
    }
  }
}

// Row tasks, one warp per 32 consecutive rows, edge-parallel: the warp walks
// its rows' cross in-edges in chunks of 256 (coalesced index loads, all the
// rank/deg gathers of a chunk in flight together), each lane computes its
// edges' terms (c * r_src) / deg_src into a warp-private stage, and the lane
// owning a row adds that row's terms in order, carrying its sum across
// chunks -- the reference's order, bit-exact, for every row.  Rows above
// kCrossSplit (= kCrossLight) are done by k_pull_heavy; a warp whose rows carry
// more than kTiledCrossMax edges takes the per-row path.
constexpr int kTiledCrossMax = 2048;

// rows [rb, re), re - rb <= 32, by the calling warp.  mode 0: whole rows;
// kTaskRowsPart: only the terms of sources in rows below `split`, the partial
// sum stored in xpart; kTaskRowsFin: xpart plus the remaining terms.  Every
// row owner adds its terms in list order, so the split changes no rounding.
template <int mode = 0>
__device__ void cross_warp_rows(const DeviceLayout& L, int rb, int re, const double* __restrict__ w, double c,
                                const double* __restrict__ pf, double* rank, double* s0, double* stage,
                                int split = 0, double* xpart = nullptr) {
  const int lane = threadIdx.x & 31;
  const int row = rb + lane;
  const bool mine = row < re;
  long long lo = 0, hi = 0;
  if (mine) {
    lo = L.xptr[row];
    hi = L.xptr[row + 1];
  }
  long long base = __shfl_sync(0xffffffffu, lo, 0);
  long long end = L.xptr[re];
  if constexpr (mode == 0)
    if (end - base > kTiledCrossMax) {
      cross_rows(L, rb, re, w, c, pf, rank, s0, lane, 32);
      return;
    }
  const bool light = mine && hi - lo <= kCrossLight;  // heavier rows: k_pull_heavy
  if constexpr (mode != 0) {  // this pass covers [lo, cut) or [cut, hi) of each row
    long long cut = lo;
    if (light)
      while (cut < hi && L.xsrc[cut] < split) ++cut;
    if constexpr (mode == kTaskRowsPart) hi = cut;
    else lo = cut;
    base = light ? lo : LLONG_MAX;  // the warp's edge window: every light row's range
    end = light ? hi : LLONG_MIN;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      base = min(base, __shfl_xor_sync(0xffffffffu, base, o));
      end = max(end, __shfl_xor_sync(0xffffffffu, end, o));
    }
  }
  double acc = 0.0;
  if (light) {
    if constexpr (mode == kTaskRowsFin) acc = xpart[row];
    else acc = w[L.vertex_of[row]];
  }
  // the finish's per-row operands, loaded now (off the gather chain)
  std::uint8_t kind = 0, lp = 0;
  int dg = 1;
  double pfr = 0.0;
  if (light) {
    kind = L.rowkind[row];
    lp = L.loop[row];
    dg = L.deg[row];
    pfr = pf[row];
  }
  for (long long cb = base; cb < end; cb += kTileNnzCross) {
    const int n = static_cast<int>(min(static_cast<long long>(kTileNnzCross), end - cb));
    int src[kTileNnzCross / 32];
#pragma unroll
    for (int k = 0; k < kTileNnzCross / 32; ++k) {
      const int e = lane + 32 * k;
      src[k] = e < n ? __ldg(L.xsrc + cb + e) : 0;
      LR_DCHECK(src[k] >= 0 && src[k] < L.n);
    }
    double rv[kTileNnzCross / 32];
    int dv[kTileNnzCross / 32];
#pragma unroll
    for (int k = 0; k < kTileNnzCross / 32; ++k) {
      rv[k] = rank[src[k]];
      dv[k] = __ldg(L.deg + src[k]);
    }
#pragma unroll
    for (int k = 0; k < kTileNnzCross / 32; ++k) {
      const int e = lane + 32 * k;
      if (e < n) stage[e] = c * rv[k] / static_cast<double>(dv[k]);
    }
    __syncwarp();
    if (light) {
      const int a = static_cast<int>(max(lo, cb) - cb), b = static_cast<int>(min(hi, cb + n) - cb);
      for (int e = a; e < b; ++e) acc += stage[e];
    }
    __syncwarp();
  }
  if constexpr (mode == kTaskRowsPart) {
    if (light) xpart[row] = acc;
  } else if (light) {  // row_finish with the prefetched operands
    if (kind == kSingle && lp) acc /= 1.0 - c / static_cast<double>(dg);
    rank[row] = acc;
    if (kind == kLargeGrid) s0[row] = pfr * acc;
  }
}

// a row task: 32 rows per warp of the CTA
template <int mode = 0>
__device__ void cross_rows_tiled(const DeviceLayout& L, int r0, int r1, const double* __restrict__ w, double c,
                                 const double* __restrict__ pf, double* rank, double* s0, double* stage,
                                 int split = 0, double* xpart = nullptr) {
  const int rb = r0 + 32 * static_cast<int>(threadIdx.x >> 5);
  if (rb < r1) cross_warp_rows<mode>(L, rb, min(rb + 32, r1), w, c, pf, rank, s0, stage, split, xpart);
}

// The start weights of a unit's rows [r0, r1) by a whole CTA of `nwarps` warps
// before it solves the unit: warp-tiled as above (32 rows per warp and round,
// every gather of a chunk in flight), each warp staging in its own
// kTileNnzCross doubles of `sm`; per-thread rows when the CTA has less shared
// memory than that.
__device__ void cross_rows_cta(const DeviceLayout& L, int r0, int r1, const double* __restrict__ w, double c,
                               const double* __restrict__ pf, double* rank, double* s0, double* sm,
                               size_t smem_bytes, int nwarps) {
  if (smem_bytes < static_cast<size_t>(nwarps) * kTileNnzCross * sizeof(double)) {
    cross_rows(L, r0, r1, w, c, pf, rank, s0, threadIdx.x, 32 * nwarps);
    return;
  }
  const int warp = threadIdx.x >> 5;
  double* stage = sm + warp * kTileNnzCross;
  for (int rb = r0 + 32 * warp; rb < r1; rb += 32 * nwarps)
    cross_warp_rows(L, rb, min(rb + 32, r1), w, c, pf, rank, s0, stage);
}

// ------------------------------------------------------------------ K3
// One depth-slice row of a CAC: parents in Kahn order, then the kept-loop
// factor (solvers.cpp:61-83).
__device__ __forceinline__ double cac_row(const DeviceLayout& L, int r, double c, const double* rank, long long e0,
                                          long long e1, double acc) {
#pragma unroll 4
  for (long long e = e0; e < e1; ++e) {
    const int s = L.isrc[e];
    LR_DCHECK(s >= 0 && s < L.n);
    acc += rank[s] * c / static_cast<double>(L.deg[s]);
  }
  return acc;
}

__device__ __forceinline__ double loop_factor(const DeviceLayout& L, int r, double c, double acc) {
  return L.loop[r] ? acc / (1.0 - c / static_cast<double>(L.deg[r])) : acc;
}

// depth sweep of one CAC by a warp (kBlock = false) or a CTA (true)
template <bool kBlock>
__device__ void cac_sweep(const DeviceLayout& L, const CacTask& t, const int* __restrict__ depth_ptr, double c,
                          double* rank, int tid, int width) {
  const int lane = threadIdx.x & 31;
  const int wid = tid >> 5, nw = width >> 5;
  const int* dp = depth_ptr + t.depth_begin;
  for (int d = 0; d < t.ndepth; ++d) {
    if (d > 0) {
      if (kBlock) {
        __syncthreads();
      } else {
        __threadfence_block();
        __syncwarp();
      }
    }
    const int s0 = dp[d], s1 = dp[d + 1];
    for (int r = s0 + tid; r < s1; r += width) {
      const long long e0 = L.iptr[r], e1 = L.iptr[r + 1];
      if (e1 - e0 > kCrossLight) continue;
      rank[r] = loop_factor(L, r, c, cac_row(L, r, c, rank, e0, e1, rank[r]));
    }
    for (int base = s0 + wid * 32; base < s1; base += nw * 32) {
      const int r = base + lane;
      long long deg_in = 0;
      if (r < s1) deg_in = L.iptr[r + 1] - L.iptr[r];
      unsigned mask = __ballot_sync(0xffffffffu, deg_in > kCrossLight);
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const int row = base + src;
        double y = 0.0;
        for (long long e = L.iptr[row] + lane; e < L.iptr[row + 1]; e += 32) {
          const int s = L.isrc[e];
          y += rank[s] * c / static_cast<double>(L.deg[s]);
        }
        y = warp_sum(y);
        if (lane == 0) rank[row] = loop_factor(L, row, c, rank[row] + y);
      }
    }
  }
}

// The same sweep with the CAC staged in shared memory: its start weights,
// row pointers, parents (as offsets into the CAC) and walk degrees are loaded
// once, all independent loads in flight together; every depth slice then
// reads only shared memory, so a slice costs a barrier instead of three
// dependent global round trips.  A finished row writes its rank to global
// memory and replaces its start weight in `sr` with the term it pushes,
// (r * c) / deg -- the exact value cac_row computes per in-edge -- so a child's
// in-edge costs two shared loads and an add, with no FP64 division on the
// slice-to-slice chain.  Same terms, same order (bit-exact).
template <bool kBlock>
__device__ void cac_sweep_staged(const DeviceLayout& L, const CacTask& t, const int* __restrict__ depth_ptr, double c,
                                 double* rank, int tid, int width, void* stage) {
  const int lane = threadIdx.x & 31;
  const int wid = tid >> 5, nw = width >> 5;
  const int rb = t.row_begin, m = t.row_end - t.row_begin;
  const long long eb = L.iptr[rb];
  const int ne = static_cast<int>(L.iptr[t.row_end] - eb);
  double* sr = static_cast<double*>(stage);
  int* rp = reinterpret_cast<int*>(sr + m);
  int* rd = rp + m + 1;  // walk out-degree of every row (parents are rows of the CAC)
  int* es = rd + m;
  std::uint8_t* lp = reinterpret_cast<std::uint8_t*>(es + ne);  // kept self-loop flags
  // staging: four rows / in-edges per thread in flight, no dependent loads
  for (int i0 = tid; i0 < m; i0 += 4 * width) {
    double rv[4];
    long long pv[4];
    int dv[4];
    std::uint8_t fv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = min(i0 + q * width, m - 1);
      rv[q] = rank[rb + i];
      pv[q] = __ldg(L.iptr + rb + i);
      dv[q] = __ldg(L.deg + rb + i);
      fv[q] = __ldg(L.loop + rb + i);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + q * width;
      if (i < m) {
        sr[i] = rv[q];
        rp[i] = static_cast<int>(pv[q] - eb);
        rd[i] = dv[q];
        lp[i] = fv[q];
      }
    }
  }
  if (tid == 0) rp[m] = ne;
  for (int e0 = tid; e0 < ne; e0 += 4 * width) {
    int sv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) sv[q] = __ldg(L.isrc + eb + min(e0 + q * width, ne - 1));
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (e0 + q * width < ne) es[e0 + q * width] = sv[q] - rb;
  }
  auto sync = [&] {
    if (kBlock) {
      __syncthreads();
    } else {
      __syncwarp();
    }
  };
  // slice bounds: dp[d + 1] is the next slice's start, so only one new bound
  // per slice, loaded a slice ahead (off the barrier-to-barrier chain)
  const int* dp = depth_ptr + t.depth_begin;
  const int nd = t.ndepth;
  int b0 = __ldg(dp) - rb, b1 = nd > 0 ? __ldg(dp + 1) - rb : b0;
  sync();
  for (int d = 0; d < nd; ++d) {
    if (d > 0) sync();
    const int s0 = b0, s1 = b1;
    if (d + 1 < nd) {
      b0 = s1;
      b1 = __ldg(dp + d + 2) - rb;
    }
    // rows of this slice: sr[i] holds the start weight, sr[parent] the
    // parent's pushed term
    auto finish = [&](int i, double acc) {
      const double dg = static_cast<double>(rd[i]);
      const double fin = lp[i] ? acc / (1.0 - c / dg) : acc;
      rank[rb + i] = fin;
      sr[i] = fin * c / dg;
    };
    for (int i = s0 + tid; i < s1; i += width) {
      const int e0 = rp[i], e1 = rp[i + 1];
      if (e1 - e0 > kCrossLight) continue;
      double acc = sr[i];
      for (int e = e0; e < e1; ++e) {
        const int sp = es[e];
        LR_DCHECK(sp >= 0 && sp < m);
        acc += sr[sp];
      }
      finish(i, acc);
    }
    for (int base = s0 + wid * 32; base < s1; base += nw * 32) {
      const int i = base + lane;
      const int deg_in = i < s1 ? rp[i + 1] - rp[i] : 0;
      unsigned mask = __ballot_sync(0xffffffffu, deg_in > kCrossLight);
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const int row = base + src;
        double y = 0.0;
        for (int e = rp[row] + lane; e < rp[row + 1]; e += 32) y += sr[es[e]];
        y = warp_sum(y);
        if (lane == 0) finish(row, sr[row] + y);
      }
    }
  }
  sync();  // the stage is free for the caller's next task
}

// CACs too large for cac_sweep_staged (k_cac_big, up to 65535 rows): only the
// structure is staged -- row offsets and 16-bit parent offsets -- and every
// finished row publishes its pushed term (r * c) / deg once to `pv` (global,
// indexed like rank), so a row of the next slice adds those terms in the same
// order as cac_row (bit-exact) with one global round trip on the chain instead
// of four.
__device__ void cac_sweep_compact(const DeviceLayout& L, const CacTask& t, const int* __restrict__ depth_ptr, double c,
                                  double* rank, double* pv, void* stage) {
  const int tid = threadIdx.x, width = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = width >> 5;
  const int rb = t.row_begin, m = t.row_end - t.row_begin;
  const long long eb = L.iptr[rb];
  const int ne = static_cast<int>(L.iptr[t.row_end] - eb);
  int* rp = static_cast<int*>(stage);
  unsigned short* es = reinterpret_cast<unsigned short*>(rp + m + 1);
  for (int i0 = tid; i0 < m; i0 += 4 * width) {
    long long o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = __ldg(L.iptr + rb + min(i0 + q * width, m - 1));
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (i0 + q * width < m) rp[i0 + q * width] = static_cast<int>(o[q] - eb);
  }
  if (tid == 0) rp[m] = ne;
  for (int e0 = tid; e0 < ne; e0 += 8 * width) {
    int v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __ldg(L.isrc + eb + min(e0 + q * width, ne - 1));
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (e0 + q * width < ne) es[e0 + q * width] = static_cast<unsigned short>(v[q] - rb);
  }
  __syncthreads();
  const double* pvb = pv + rb;
  auto finish = [&](int i, double acc) {
    const int r = rb + i;
    const double dg = static_cast<double>(__ldg(L.deg + r));
    const double fin = __ldg(L.loop + r) ? acc / (1.0 - c / dg) : acc;
    rank[r] = fin;
    pv[r] = fin * c / dg;
  };
  const int* dp = depth_ptr + t.depth_begin;
  for (int d = 0; d < t.ndepth; ++d) {
    if (d > 0) __syncthreads();
    const int s0 = dp[d] - rb, s1 = dp[d + 1] - rb;
    for (int i = s0 + tid; i < s1; i += width) {
      const int e0 = rp[i], e1 = rp[i + 1];
      if (e1 - e0 > kCrossLight) continue;
      double acc = rank[rb + i];
      for (int e = e0; e < e1; ++e) acc += pvb[es[e]];
      finish(i, acc);
    }
    for (int base = s0 + wid * 32; base < s1; base += nw * 32) {
      const int i = base + lane;
      const int deg_in = i < s1 ? rp[i + 1] - rp[i] : 0;
      unsigned mask = __ballot_sync(0xffffffffu, deg_in > kCrossLight);
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const int row = base + src;
        double y = 0.0;
        for (int e = rp[row] + lane; e < rp[row + 1]; e += 32) y += pvb[es[e]];
        y = warp_sum(y);
        if (lane == 0) finish(row, rank[rb + row] + y);
      }
    }
  }
}

__host__ __device__ constexpr size_t cac_compact_bytes(long long m, long long ne) {
  return static_cast<size_t>(m + 1) * 4 + static_cast<size_t>(ne) * 2 + 16;
}

// bytes cac_sweep_staged needs for a CAC of m rows and ne in-edges
__host__ __device__ constexpr size_t cac_stage_bytes(long long m, long long ne) {
  return static_cast<size_t>(m) * 13 + static_cast<size_t>(m + 1) * 4 + static_cast<size_t>(ne) * 4 + 16;
}

// ------------------------------------------------------------------ K5
// Dense (I - cA^T) r = w per SccSmall unit in shared memory
// (solve_dense_system, solvers.cpp:92-108).  The matrix is strictly
// diagonally dominant by columns (column sums of cA^T <= c < 1), so partial
// pivoting never swaps and plain elimination equals the reference's LU.
// One barrier per elimination step; back substitution by one warp.
__device__ void small_solve(const DeviceLayout& L, const SccTask& t, int ld, const double* __restrict__ pf,
                            double* rank, double* sm, double* red, DevStatus* st) {
  double* M = sm;
  double* rhs = M + static_cast<size_t>(ld) * ld;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rb = t.row_begin, m = t.row_end - t.row_begin;
  for (int i = tid; i < m * ld; i += kThreads) M[i] = 0.0;
  __syncthreads();
  for (int b = tid; b < m; b += kThreads) {
    M[b * ld + b] = 1.0;
    rhs[b] = rank[rb + b];
  }
  __syncthreads();
  for (int b = tid; b < m; b += kThreads) {
    const long long e1 = L.iptr[rb + b + 1];
    for (long long e = L.iptr[rb + b]; e < e1; ++e) {
      const int s = L.isrc[e];
      M[b * ld + (s - rb)] -= pf[s];
    }
  }
  // Gauss-Jordan: one barrier per pivot, no back substitution.  Each warp
  // owns rows i = warp (mod 8) and takes them 8 at a time, so the 8 row
  // factors are loaded together and the column updates of 8 rows overlap.
  for (int k = 0; k < m; ++k) {
    __syncthreads();
    const double inv = 1.0 / M[k * ld + k];
    const double rk = rhs[k];
    for (int i0 = warp; i0 < m; i0 += 8 * kWarpsPer) {
      double f[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * kWarpsPer;
        f[u] = (i < m && i != k) ? M[i * ld + k] * inv : 0.0;
      }
      if (lane == 0) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * kWarpsPer;
          if (i < m && i != k) rhs[i] -= f[u] * rk;
        }
      }
      for (int j = k + 1 + lane; j < m; j += 32) {
        const double pkj = M[k * ld + j];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * kWarpsPer;
          if (i < m && i != k) M[i * ld + j] -= f[u] * pkj;
        }
      }
    }
  }
  __syncthreads();
  for (int b = tid; b < m; b += kThreads) rhs[b] /= M[b * ld + b];
  __syncthreads();
  // residual check of solvers.cpp:103-106
  double res = 0.0, wm = 0.0, xm = 0.0;
  for (int b = tid; b < m; b += kThreads) {
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
  for (int b = tid; b < m; b += kThreads) rank[rb + b] = rhs[b];
}

// Gauss-Jordan for m <= kSmallTileMaxM, shaped for the per-step latency
// (measured on B200: FP64 multiply/add 23 cycles, shared load 29, barrier 38,
// IEEE double division 90 -- the chain of dependent operations per
// elimination step is what the solve time is made of).
//  * The system [I - cA^T | w] is an m x (m+1) tile with an odd row stride;
//    thread (warp, lane) always owns rows lane + 32a and columns warp + 8b.
//  * Fraction-free (Bareiss) Gauss-Jordan: step k replaces every row i != k by
//    (p_k * row_i - M[i][k] * row_k) * r, r ~ 1/p_{k-1}, on the columns j > k.
//    The entries stay near minors of the matrix, within [(1-c)^m, (1+c)^m];
//    r comes from the hardware reciprocal approximation issued in step k-1,
//    so a step's chain is shared load -> two multiplies -> multiply pair ->
//    subtract -> store, without a division.  The step reads column k and
//    row k and writes neither: one barrier per step.  Finished rows keep
//    their diagonal in step with the others (the owner of M[i][i] applies
//    p_k / p_{k-1}), so x_i = M[i][m] / M[i][i] at the end.
//  * The in-edges are stashed in shared memory during assembly so the
//    residual check of solvers.cpp:103-106 needs no second global gather.
#ifdef LR_TILE_PROBE
__device__ long long* g_tile_probe;
#endif
#ifndef LR_SMALL_PAIR
#define LR_SMALL_PAIR 1
#endif
template <int A>
__device__ void small_solve_tile(const DeviceLayout& L, const SccTask& t, const double* __restrict__ pf,
                                 double* rank, double* sm, unsigned long long* red, DevStatus* st) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rb = t.row_begin, m = t.row_end - t.row_begin;
  const int ld = small_tile_ld(m);  // zero columns past m: a chunk never needs a bound check
  const long long eb = L.iptr[rb];
  const int ne = static_cast<int>(L.iptr[t.row_end] - eb);
  double* M = sm;
  double* x = M + static_cast<size_t>(m) * ld;
  double* ev = x + m;
  int* es = reinterpret_cast<int*>(ev + ne);
  // this thread's row (m <= kThreads): start weight and in-edge range, loaded
  // before the tile is cleared so the global latency overlaps it
  const bool mine = tid < m;
  double wb = 0.0;
  int e0 = 0, e1 = 0;
  if (mine) {
    wb = rank[rb + tid];
    e0 = static_cast<int>(L.iptr[rb + tid] - eb);
    e1 = static_cast<int>(L.iptr[rb + tid + 1] - eb);
  }
  for (int i = tid; i < m * ld; i += kThreads) M[i] = 0.0;
  __syncthreads();
  if (mine) {
    double* Mr = M + static_cast<size_t>(tid) * ld;
    Mr[tid] = 1.0;
    Mr[m] = wb;
    for (int e = e0; e < e1; ++e) {
      const int s = L.isrc[eb + e];
      const double v = pf[s];
      es[e] = s - rb;
      ev[e] = v;
      Mr[s - rb] -= v;
    }
  }
  double* row[A];
  bool valid[A], diag[A];
#pragma unroll
  for (int a = 0; a < A; ++a) {
    const int i = lane + 32 * a;
    valid[a] = i < m;
    diag[a] = valid[a] && (i & 7) == warp;  // this thread owns M[i][i]
    row[a] = M + static_cast<size_t>(valid[a] ? i : 0) * ld;
  }
  double rprev = 1.0;  // 1 / p_{k-1}
  int k0 = 0;
#if LR_SMALL_PAIR
  // Two pivots per pass (the shared-memory port is the bound: one load and one
  // store per trailing entry per pass instead of per pivot).  Phase A updates
  // only row k+1 (columns > k) and column k+1 (rows other than k, k+1) with
  // pivot k, one entry per thread; phase B applies both pivots to every other
  // entry right of column k+1 in registers:
  //   i != k:  (pp1 (pp0 v - f0 T[k][j]) - f1 T'[k+1][j])
  //   i == k:  pp1 v - f1 T[k][j]... (row k is pivot k's row: only pivot k+1 acts)
  // with the same fraction-free scaling as the single step below.
  for (; k0 + 1 < m; k0 += 2) {
    const int k = k0;
    __syncthreads();
    const double* pr0 = M + static_cast<size_t>(k) * ld;
    double* pr1 = M + static_cast<size_t>(k + 1) * ld;
    const double p0 = pr0[k];
    const double pp0 = p0 * rprev;
    double r1;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r1) : "d"(p0));
    {  // phase A
      const int j = k + 1 + tid;
      if (j <= m) pr1[j] = __fma_rn(-(pr1[k] * rprev), pr0[j], pp0 * pr1[j]);
      if (tid < m && tid != k && tid != k + 1) {
        double* Ti = M + static_cast<size_t>(tid) * ld;
        Ti[k + 1] = __fma_rn(-(Ti[k] * rprev), pr0[k + 1], pp0 * Ti[k + 1]);
      }
    }
    __syncthreads();
    const double p1 = pr1[k + 1];
    const double pp1 = p1 * r1;
    double f0[A], f1[A];
    bool ok[A], isk[A];
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int i = lane + 32 * a;
      f0[a] = row[a][k] * rprev;
      f1[a] = row[a][k + 1] * r1;
      isk[a] = i == k;
      ok[a] = valid[a] && i != k + 1;
    }
    for (int j = warp + ((k + 9 - warp) & ~7); j <= m; j += 32) {
      double pa[4], pb[4], v[4][A];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        pa[q] = pr0[j + 8 * q];
        pb[q] = pr1[j + 8 * q];
#pragma unroll
        for (int a = 0; a < A; ++a) v[q][a] = row[a][j + 8 * q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int a = 0; a < A; ++a) {
          const double u = isk[a] ? v[q][a] : __fma_rn(-f0[a], pa[q], pp0 * v[q][a]);
          v[q][a] = __fma_rn(-f1[a], pb[q], pp1 * u);
        }
#pragma unroll
      for (int a = 0; a < A; ++a)
        if (ok[a]) {
#pragma unroll
          for (int q = 0; q < 4; ++q) row[a][j + 8 * q] = v[q][a];
        }
    }
#pragma unroll
    for (int a = 0; a < A; ++a) {  // finished rows: the diagonal follows the row scales
      const int i = lane + 32 * a;
      if (diag[a] && i < k) row[a][i] *= pp0 * pp1;
      if (diag[a] && i == k) row[a][i] *= pp1;
    }
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rprev) : "d"(p1));
  }
#endif
  for (int k = k0; k < m; ++k) {
    __syncthreads();
#ifdef LR_TILE_PROBE  // tools/small_bench.cu: per-step cycle stamps of warp 0
    if (threadIdx.x == 0) g_tile_probe[blockIdx.x * 160 + k] = clock64();
#endif
    const double* pr = M + static_cast<size_t>(k) * ld;
    const double p = pr[k];
    const double pp = p * rprev;
    double f[A];
    bool ok[A];
#pragma unroll
    for (int a = 0; a < A; ++a) {
      f[a] = row[a][k] * rprev;
      ok[a] = valid[a] && lane + 32 * a != k;
    }
    // first owned column above k, then four owned columns per chunk: all
    // loads first, then the updates, then the stores (columns past m are zero
    // padding and stay zero)
    for (int j = warp + ((k + 8 - warp) & ~7); j <= m; j += 32) {
      double pk[4], v[4][A];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        pk[q] = pr[j + 8 * q];
#pragma unroll
        for (int a = 0; a < A; ++a) v[q][a] = row[a][j + 8 * q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int a = 0; a < A; ++a) v[q][a] = __fma_rn(-f[a], pk[q], pp * v[q][a]);  // one rounding fewer than the
#pragma unroll                                                                       // reference's LU: not bit-exact anyway
      for (int a = 0; a < A; ++a)
        if (ok[a]) {
#pragma unroll
          for (int q = 0; q < 4; ++q) row[a][j + 8 * q] = v[q][a];
        }
    }
#pragma unroll
    for (int a = 0; a < A; ++a)  // finished rows: the diagonal follows the row scale
      if (diag[a] && lane + 32 * a < k) row[a][lane + 32 * a] *= pp;
    // Row scale for step k+1.  Any nonzero factor is a valid row operation
    // (the solution does not depend on it); ~1/p_k only keeps the entries
    // near the minors, so the hardware approximation (one MUFU, no Newton
    // steps, no branch) is enough.
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rprev) : "d"(p));
  }
  __syncthreads();
  double xb = 0.0;
  if (mine) {
    xb = M[static_cast<size_t>(tid) * ld + m] / M[static_cast<size_t>(tid) * ld + tid];
    x[tid] = xb;
  }
  __syncthreads();
  // residual check of solvers.cpp:103-106 on the stashed in-edges; maxima of
  // non-negative doubles as integer maxima of their bit patterns
  unsigned long long res = 0, wm = 0, xm = 0;
  if (mine) {
    double acc = xb;
    for (int e = e0; e < e1; ++e) acc -= ev[e] * x[es[e]];
    res = dbits(fabs(acc - wb));
    wm = dbits(fabs(wb));
    xm = dbits(fabs(xb));
    rank[rb + tid] = xb;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    res = max(res, __shfl_xor_sync(0xffffffffu, res, o));
    wm = max(wm, __shfl_xor_sync(0xffffffffu, wm, o));
    xm = max(xm, __shfl_xor_sync(0xffffffffu, xm, o));
  }
  if (lane == 0) {
    red[warp] = res;
    red[8 + warp] = wm;
    red[16 + warp] = xm;
  }
  __syncthreads();
  if (tid == 0) {
    for (int i = 1; i < kWarpsPer; ++i) {
      res = max(res, red[i]);
      wm = max(wm, red[8 + i]);
      xm = max(xm, red[16 + i]);
    }
    if (!(bitsd(res) <= 1e-8 * (1.0 + bitsd(wm) + bitsd(xm)))) atomicOr(&st->err, kErrDegen);
  }
}

// ------------------------------------------------------------------ K5b
// SccSmall units of up to 64 rows: block Gauss-Jordan on 8 x 8 tiles with the
// FP64 tensor cores (DMMA m8n8k4).  The system [I - cA^T | w], padded to
// 64 x 72 (rows and columns past m: identity; the right-hand side in column
// 64), lives in the accumulators: warp w holds row tile w, nine column tiles
// of two doubles per lane, for the whole solve.  Block step k: warp k's row
// block R and every warp's column block C go to shared memory, every warp
// inverts the 8 x 8 pivot block P (strictly diagonally dominant by columns:
// no pivoting) in registers, R' = P^-1 R (DMMA), and every other row tile
// takes the rank-8 update -= C R' (18 DMMA per warp); row tile k becomes R'.
// Shared-memory traffic per step is the two blocks, not the trailing matrix,
// so eight steps replace 64 port-bound pivots.  Not bit-exact (the reference's
// LU differs by rounding): the residual check of solvers.cpp:103-106 follows.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// One row of a small system: its in-edges' columns and pf values stashed for
// the residual check and subtracted from the row (each column once), four
// in-edges' index and pf loads in flight at a time.
__device__ __forceinline__ void stage_row_edges(const DeviceLayout& L, const double* __restrict__ pf, int rb,
                                                long long eb, int e0, int e1, int* es, double* ev, double* Mr) {
  for (int e = e0; e < e1; e += 4) {
    int sv[4];
    double pv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) sv[q] = __ldg(L.isrc + eb + min(e + q, e1 - 1));
#pragma unroll
    for (int q = 0; q < 4; ++q) pv[q] = pf[sv[q]];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (e + q < e1) {
        es[e + q] = sv[q] - rb;
        ev[e + q] = pv[q];
        Mr[sv[q] - rb] -= pv[q];
      }
  }
}

// The inverse of an 8 x 8 pivot block by Gauss-Jordan on [P | I] in
// registers (no pivoting: the blocks are strictly diagonally dominant by
// columns).  Lane (g, tq) holds P[g][2tq], P[g][2tq+1]; returns its A fragments
// of P^-1 for DMMA m8n8k4 (row g, columns tq and 4 + tq).
// Division-free elimination: step pv replaces row g != pv by
// piv * row_g - P[g][pv] * row_pv (any nonzero multiple of a row is a valid row
// operation), which leaves the pivot row alone and keeps the reciprocal off the
// eight-step dependent chain (shuffle + multiply + fma per step instead of
// shuffle + reciprocal + two Newton steps + multiply + fma: ~190 -> ~80 cycles).
// The left block ends up diagonal; each row is divided by its diagonal entry
// once at the end (eight independent reciprocals).  Entries scale by at most the
// product of the pivots, which lie in (1 - c, 1 + c): no overflow in 8 steps.
__device__ __forceinline__ void pivot_block_inverse(double p0, double p1, int g, int tq, double& ia, double& ib) {
  double q0 = g == 2 * tq ? 1.0 : 0.0, q1 = g == 2 * tq + 1 ? 1.0 : 0.0;
#pragma unroll
  for (int pv = 0; pv < 8; ++pv) {
    const int src = pv * 4 + tq;  // row pv, my columns
    const double rp0 = __shfl_sync(0xffffffffu, p0, src), rp1 = __shfl_sync(0xffffffffu, p1, src);
    const double rq0 = __shfl_sync(0xffffffffu, q0, src), rq1 = __shfl_sync(0xffffffffu, q1, src);
    const double piv = __shfl_sync(0xffffffffu, (pv & 1) ? p1 : p0, pv * 4 + (pv >> 1));
    const double f = __shfl_sync(0xffffffffu, (pv & 1) ? p1 : p0, g * 4 + (pv >> 1));  // P[g][pv]
    if (g != pv) {
      p0 = __fma_rn(piv, p0, -(f * rp0));
      p1 = __fma_rn(piv, p1, -(f * rp1));
      q0 = __fma_rn(piv, q0, -(f * rq0));
      q1 = __fma_rn(piv, q1, -(f * rq1));
    }
  }
  // 1 / P[g][g]: hardware reciprocal plus two Newton steps (~1 ulp)
  const double dg = __shfl_sync(0xffffffffu, (g & 1) ? p1 : p0, g * 4 + (g >> 1));
  double inv;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(dg));
  inv = __fma_rn(inv, __fma_rn(-dg, inv, 1.0), inv);
  inv = __fma_rn(inv, __fma_rn(-dg, inv, 1.0), inv);
  q0 *= inv;
  q1 *= inv;
  const double u0 = __shfl_sync(0xffffffffu, q0, g * 4 + (tq >> 1)), u1 = __shfl_sync(0xffffffffu, q1, g * 4 + (tq >> 1));
  const double v0 = __shfl_sync(0xffffffffu, q0, g * 4 + 2 + (tq >> 1)),
               v1 = __shfl_sync(0xffffffffu, q1, g * 4 + 2 + (tq >> 1));
  ia = (tq & 1) ? u1 : u0;
  ib = (tq & 1) ? v1 : v0;
}

__device__ void small_solve_mma(const DeviceLayout& L, const SccTask& t, const double* __restrict__ pf,
                                double* rank, double* sm, unsigned long long* red, DevStatus* st) {
  constexpr int W = 72;  // columns of the padded system (9 tiles)
  static_assert(kWarpsPer == 8, "one 8-row tile per warp");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;  // fragment row / column pair
  const int rb = t.row_begin, m = t.row_end - t.row_begin;
  const long long eb = L.iptr[rb];
  const int ne = static_cast<int>(L.iptr[t.row_end] - eb);
  double* M = sm;           // 64 x 72 build area, then the step buffers
  double* x = M + 64 * W;   // solution
  double* ev = x + 64;      // in-edge values and columns (residual check)
  int* es = reinterpret_cast<int*>(ev + ne);
  const bool mine = tid < m;
  double wb = 0.0;
  int e0 = 0, e1 = 0;
  if (mine) {
    wb = rank[rb + tid];
    e0 = static_cast<int>(L.iptr[rb + tid] - eb);
    e1 = static_cast<int>(L.iptr[rb + tid + 1] - eb);
  }
  for (int r = warp; r < 64; r += kWarpsPer)  // identity (no integer division per entry)
    for (int cidx = lane; cidx < W; cidx += 32) M[r * W + cidx] = cidx == r ? 1.0 : 0.0;
  __syncthreads();
  if (mine) {
    double* Mr = M + tid * W;
    Mr[64] = wb;
    stage_row_edges(L, pf, rb, eb, e0, e1, es, ev, Mr);
  }
  __syncthreads();
  double acc[9][2];
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    acc[j][0] = M[(8 * warp + g) * W + 8 * j + 2 * tq];
    acc[j][1] = M[(8 * warp + g) * W + 8 * j + 2 * tq + 1];
  }
  double* Rb = M;            // 8 x 72: pivot row block
  double* Cb = M + 8 * W;    // 64 x 8: pivot column block
  double* Rp = Cb + 64 * 8;  // 8 x 72: P^-1 R
  const int nb = (m + 7) >> 3;
  for (int kb = 0; kb < nb; ++kb) {
    __syncthreads();  // the previous step's readers of Rb / Cb / Rp are done
    if (warp == kb) {
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        Rb[g * W + 8 * j + 2 * tq] = acc[j][0];
        Rb[g * W + 8 * j + 2 * tq + 1] = acc[j][1];
      }
    }
    {  // column block kb of this row tile (acc[kb], kb warp-uniform)
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j == kb) {
          c0 = acc[j][0];
          c1 = acc[j][1];
        }
      Cb[(8 * warp + g) * 8 + 2 * tq] = c0;
      Cb[(8 * warp + g) * 8 + 2 * tq + 1] = c1;
    }
    __syncthreads();
    // P^-1 (A fragments: row g, columns tq and 4 + tq)
    double ia, ib;
    pivot_block_inverse(Rb[g * W + 8 * kb + 2 * tq], Rb[g * W + 8 * kb + 2 * tq + 1], g, tq, ia, ib);
    // R' = P^-1 R: column tile `warp` (and tile 8 by warp 0)
    for (int j = warp; j < 9; j += kWarpsPer) {
      double d0 = 0.0, d1 = 0.0;
      dmma(d0, d1, ia, Rb[tq * W + 8 * j + g]);
      dmma(d0, d1, ib, Rb[(4 + tq) * W + 8 * j + g]);
      Rp[g * W + 8 * j + 2 * tq] = d0;
      Rp[g * W + 8 * j + 2 * tq + 1] = d1;
    }
    __syncthreads();
    if (warp == kb) {
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        acc[j][0] = Rp[g * W + 8 * j + 2 * tq];
        acc[j][1] = Rp[g * W + 8 * j + 2 * tq + 1];
      }
    } else {
      const double a0 = -Cb[(8 * warp + g) * 8 + tq], a1 = -Cb[(8 * warp + g) * 8 + 4 + tq];
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        dmma(acc[j][0], acc[j][1], a0, Rp[tq * W + 8 * j + g]);
        dmma(acc[j][0], acc[j][1], a1, Rp[(4 + tq) * W + 8 * j + g]);
      }
    }
  }
  // x = column 64 (the pivot blocks are now I up to rounding)
  if (tq == 0 && 8 * warp + g < m) x[8 * warp + g] = acc[8][0];
  __syncthreads();
  unsigned long long res = 0, wm = 0, xm = 0;
  if (mine) {
    const double xb = x[tid];
    double acc_r = xb;
    for (int e = e0; e < e1; ++e) acc_r -= ev[e] * x[es[e]];
    res = dbits(fabs(acc_r - wb));
    wm = dbits(fabs(wb));
    xm = dbits(fabs(xb));
    rank[rb + tid] = xb;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    res = max(res, __shfl_xor_sync(0xffffffffu, res, o));
    wm = max(wm, __shfl_xor_sync(0xffffffffu, wm, o));
    xm = max(xm, __shfl_xor_sync(0xffffffffu, xm, o));
  }
  if (lane == 0) {
    red[warp] = res;
    red[8 + warp] = wm;
    red[16 + warp] = xm;
  }
  __syncthreads();
  if (tid == 0) {
    for (int i = 1; i < kWarpsPer; ++i) {
      res = max(res, red[i]);
      wm = max(wm, red[8 + i]);
      xm = max(xm, red[16 + i]);
    }
    if (!(bitsd(res) <= 1e-8 * (1.0 + bitsd(wm) + bitsd(xm)))) atomicOr(&st->err, kErrDegen);
  }
}

// SccSmall units of 65..kSmallMmaSmemMaxM rows: the same block Gauss-Jordan
// with the system in shared memory (mp x (mp + 8), mp = m rounded up to 8, the
// right-hand side in column mp): per block step every 8 x 8 tile is read and
// written once (2 DMMA in between), a quarter of the paired-pivot tile solve's
// traffic, and ceil(m/8) pivot-block chains instead of m pivots.
__device__ void small_solve_mma_smem(const DeviceLayout& L, const SccTask& t, const double* __restrict__ pf,
                                     double* rank, double* sm, unsigned long long* red, DevStatus* st) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int rb = t.row_begin, m = t.row_end - t.row_begin;
  // row stride = 8 mod 16 doubles: a tile's 16-byte row pieces hit distinct bank quads
  const int mp = (m + 7) & ~7, W = mp + ((mp & 15) ? 16 : 8), nrt = mp >> 3, nct = W >> 3;
  const long long eb = L.iptr[rb];
  const int ne = static_cast<int>(L.iptr[t.row_end] - eb);
  double* M = sm;                       // mp x W system
  double* Cb = M + mp * W;              // mp x 8 pivot column block
  double* Rp = Cb + mp * 8;             // 8 x W: P^-1 R
  double* x = Rp + 8 * W;               // solution
  double* ev = x + mp;                  // in-edge values and columns (residual check)
  int* es = reinterpret_cast<int*>(ev + ne);
  const bool mine = tid < m;
  double wb = 0.0;
  int e0 = 0, e1 = 0;
  if (mine) {
    wb = rank[rb + tid];
    e0 = static_cast<int>(L.iptr[rb + tid] - eb);
    e1 = static_cast<int>(L.iptr[rb + tid + 1] - eb);
  }
  for (int r = warp; r < mp; r += kWarpsPer)
    for (int cidx = lane; cidx < W; cidx += 32) M[r * W + cidx] = cidx == r ? 1.0 : 0.0;
  __syncthreads();
  if (mine) {
    double* Mr = M + tid * W;
    Mr[mp] = wb;
    stage_row_edges(L, pf, rb, eb, e0, e1, es, ev, Mr);
  }
  for (int kb = 0; kb < nrt; ++kb) {
    __syncthreads();
    for (int i = tid; i < mp * 8; i += kThreads) Cb[i] = M[(i >> 3) * W + 8 * kb + (i & 7)];
    __syncthreads();
    double ia, ib;
    pivot_block_inverse(M[(8 * kb + g) * W + 8 * kb + 2 * tq], M[(8 * kb + g) * W + 8 * kb + 2 * tq + 1], g, tq, ia, ib);
    const double* Rb = M + 8 * kb * W;
    for (int j = warp; j < nct; j += kWarpsPer) {
      double d0 = 0.0, d1 = 0.0;
      dmma(d0, d1, ia, Rb[tq * W + 8 * j + g]);
      dmma(d0, d1, ib, Rb[(4 + tq) * W + 8 * j + g]);
      Rp[g * W + 8 * j + 2 * tq] = d0;
      Rp[g * W + 8 * j + 2 * tq + 1] = d1;
    }
    __syncthreads();
    // warp w: row tiles w, w + 8 (<= 16 row tiles), every column tile; two
    // independent DMMA chains per column tile in flight
    for (int rt0 = warp; rt0 < nrt; rt0 += 2 * kWarpsPer) {
      const int rt1 = rt0 + kWarpsPer;
      const bool has1 = rt1 < nrt;
      const double a00 = -Cb[(8 * rt0 + g) * 8 + tq], a01 = -Cb[(8 * rt0 + g) * 8 + 4 + tq];
      const double a10 = has1 ? -Cb[(8 * rt1 + g) * 8 + tq] : 0.0, a11 = has1 ? -Cb[(8 * rt1 + g) * 8 + 4 + tq] : 0.0;
      for (int ct = 0; ct < nct; ++ct) {
        const double b0 = Rp[tq * W + 8 * ct + g], b1 = Rp[(4 + tq) * W + 8 * ct + g];
        const double2 r = *reinterpret_cast<const double2*>(Rp + g * W + 8 * ct + 2 * tq);
        double2* T0 = reinterpret_cast<double2*>(M + (8 * rt0 + g) * W + 8 * ct + 2 * tq);
        double2* T1 = reinterpret_cast<double2*>(M + (8 * (has1 ? rt1 : rt0) + g) * W + 8 * ct + 2 * tq);
        double2 c = *T0, e = *T1;
        dmma(c.x, c.y, a00, b0);
        dmma(e.x, e.y, a10, b0);
        dmma(c.x, c.y, a01, b1);
        dmma(e.x, e.y, a11, b1);
        *T0 = rt0 == kb ? r : c;
        if (has1) *T1 = rt1 == kb ? r : e;
      }
    }
  }
  __syncthreads();
  if (mine) x[tid] = M[tid * W + mp];
  __syncthreads();
  unsigned long long res = 0, wm = 0, xm = 0;
  if (mine) {
    const double xb = x[tid];
    double acc_r = xb;
    for (int e = e0; e < e1; ++e) acc_r -= ev[e] * x[es[e]];
    res = dbits(fabs(acc_r - wb));
    wm = dbits(fabs(wb));
    xm = dbits(fabs(xb));
    rank[rb + tid] = xb;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    res = max(res, __shfl_xor_sync(0xffffffffu, res, o));
    wm = max(wm, __shfl_xor_sync(0xffffffffu, wm, o));
    xm = max(xm, __shfl_xor_sync(0xffffffffu, xm, o));
  }
  if (lane == 0) {
    red[warp] = res;
    red[8 + warp] = wm;
    red[16 + warp] = xm;
  }
  __syncthreads();
  if (tid == 0) {
    for (int i = 1; i < kWarpsPer; ++i) {
      res = max(res, red[i]);
      wm = max(wm, red[8 + i]);
      xm = max(xm, red[16 + i]);
    }
    if (!(bitsd(res) <= 1e-8 * (1.0 + bitsd(wm) + bitsd(xm)))) atomicOr(&st->err, kErrDegen);
  }
}

#ifndef LR_SMALL_MMA
#define LR_SMALL_MMA 1
#endif

__device__ void small_dispatch(const DeviceLayout& L, const SccTask& t, int ld, double c,
                               const double* __restrict__ pf, double* rank, double* sm, double* red, DevStatus* st) {
  const int m = t.row_end - t.row_begin;
  auto* r = reinterpret_cast<unsigned long long*>(red);
  if (LR_SMALL_MMA && m <= kSmallMmaMaxM)
    small_solve_mma(L, t, pf, rank, sm, r, st);
  else if (LR_SMALL_MMA && m <= kSmallMmaSmemMaxM)
    small_solve_mma_smem(L, t, pf, rank, sm, r, st);
  else if (!small_tile_ok(m, c))
    small_solve(L, t, ld, pf, rank, sm, red, st);
  else if (m <= 32)
    small_solve_tile<1>(L, t, pf, rank, sm, r, st);
  else if (m <= 64)
    small_solve_tile<2>(L, t, pf, rank, sm, r, st);
  else
    small_solve_tile<4>(L, t, pf, rank, sm, r, st);
}

// ------------------------------------------------------------------ K4a
// Block max of non-negative doubles as the max of their bit patterns: two
// warp reductions (high word, then low word among the lanes holding the top
// high word), one barrier, eight integer compares -- no FP64 on the chain.
__device__ __forceinline__ unsigned long long block_max_bits(unsigned long long v, unsigned long long* red) {
  const unsigned hi = static_cast<unsigned>(v >> 32);
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? static_cast<unsigned>(v) : 0u);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = (static_cast<unsigned long long>(mh) << 32) | ml;
  __syncthreads();
  // every warp reduces the per-warp maxima again: one load and two redux per lane
  const int lane = threadIdx.x & 31;
  const unsigned long long w = lane < kWarpsPer ? red[lane] : 0ull;
  const unsigned h2 = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(w >> 32));
  const unsigned l2 = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(w >> 32) == h2 ? static_cast<unsigned>(w) : 0u);
  return (static_cast<unsigned long long>(h2) << 32) | l2;
}

// Interleaved pushed vectors of lcta_solve_staged's register path: element i of
// vector b at double 32 * (i / 16) + 16 * b + i % 16 (same bank pair i % 16 in
// both, the other vector 128 bytes further).
__device__ __forceinline__ int lcta_il(int i) { return ((i >> 4) << 5) | (i & 15); }

// The whole power series of one SccLarge unit in one CTA (solve_large_scc,
// solvers.cpp:128-162), everything in shared memory: the pushed vectors, the
// ranks, pf, the row offsets and the in-edges as 16-bit offsets into the unit,
// so an iteration touches no global memory -- one thread per row, a warp for
// rows above kCrossLight, and the stop test on integer maxima.  Summation
// order is NOT the reference's source-ordered push: the register path sums a
// row's first twelve terms pairwise and the host reorders each row's in-edges
// to spread the gathers over the shared-memory banks (LR_BANK_ORDER=0 keeps
// source order), so rows agree to ~1e-16 relative; per-unit iteration counts
// equal the reference's in every parity test (run with both orders).

// pairwise sum of N terms (N a multiple of 4): log2 N dependent adds instead of N
template <int N>
__device__ __forceinline__ double tree_sum(const double* v) {
  if constexpr (N == 4) {
    return (v[0] + v[1]) + (v[2] + v[3]);
  } else if constexpr ((N & (N - 1)) == 0) {
    return tree_sum<N / 2>(v) + tree_sum<N / 2>(v + N / 2);
  } else {
    constexpr int P = N & -N;  // lowest power-of-two part
    return tree_sum<N - P>(v) + tree_sum<P>(v + N - P);
  }
}
__device__ void lcta_solve_staged(const DeviceLayout& L, const SccTask& t, int maxrows,
                                  const SolveParams* __restrict__ p, const double* __restrict__ pf, double* rank,
                                  long long* unit_iters, DevStatus* st, double* sm, double (*red)[32]) {
#ifdef LR_LCTA_PROBE
  constexpr bool kLctaProbe = true;
#else
  constexpr bool kLctaProbe = false;
#endif
  const int rb = t.row_begin, m = t.row_end - t.row_begin;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sc = sm;
  double* sn = sm + maxrows;
  double* pl = sm + 2 * maxrows;
  double* rk = sm + 3 * maxrows;
  int* rp = reinterpret_cast<int*>(sm + 4 * maxrows);
  unsigned short* es = reinterpret_cast<unsigned short*>(sm + 4 * maxrows + (maxrows + 2) / 2);
  const long long eb = L.iptr[rb];
  const int ne = static_cast<int>(L.iptr[t.row_end] - eb);
  // register rows, no warp rows: the two pushed vectors interleaved in blocks
  // of 16 (lcta_il), so the vector read in an iteration is an immediate offset
  const bool fast = m <= kLctaRegRows && !t.pad && !kLctaProbe;
  for (int i0 = threadIdx.x; i0 < m; i0 += 2 * kThreads) {  // two rows per thread in flight
    double pv[2], r[2];
    long long o[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = min(i0 + q * kThreads, m - 1);
      pv[q] = pf[rb + i];
      r[q] = rank[rb + i];
      o[q] = __ldg(L.iptr + rb + i);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = i0 + q * kThreads;
      if (i < m) {
        pl[i] = pv[q];
        rk[i] = r[q];
        sm[fast ? lcta_il(i) : i] = pv[q] * r[q];
        rp[i] = static_cast<int>(o[q] - eb);
      }
    }
  }
  if (threadIdx.x == 0) {
    rp[m] = ne;
    if (fast) sm[lcta_il(m)] = sm[lcta_il(m) + 16] = 0.0;  // the zero slot (maxrows > m) of both vectors
  }
  for (int e0 = threadIdx.x; e0 < ne; e0 += 8 * kThreads) {  // eight in-edges per thread in flight
    int v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __ldg(L.isrc + eb + min(e0 + q * kThreads, ne - 1));
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (e0 + q * kThreads < ne) es[e0 + q * kThreads] = static_cast<unsigned short>(v[q] - rb);
  }
  __syncthreads();
  const double tol = p->tol;
  const long long cap = p->cap;
  auto* rb2 = reinterpret_cast<unsigned long long(*)[32]>(red);
  long long it = 0;
  bool fail = false;
#ifdef LR_LCTA_PROBE  // tools/build_variant.sh probe: thread 0's cycles in the row phase / the stop test
  long long cyc_rows = 0, cyc_max = 0, cyc_t0 = 0, cyc_t1 = 0;
#endif
  // Units of up to 2 kThreads rows (one pass of the row loop): each thread's
  // two rows keep their loop invariants in registers across iterations -- edge
  // range, the first four in-edge offsets, pf and the rank accumulator -- so an
  // iteration's chain is the gathers of sc, the adds and the stores of sn.
  static_assert(kLctaRegRows == 2 * kThreads, "two register rows per thread");
  const bool reg_rows = m <= kLctaRegRows;
  const int ri0 = threadIdx.x, ri1 = threadIdx.x + kThreads;
  int ra0 = 0, rna = 0, rb0 = 0, rnb = 0;
  int ria[kLctaRegIdx], rib[kLctaRegIdx];
  double rpl0 = 0.0, rpl1 = 0.0, rrk0 = 0.0, rrk1 = 0.0;
  bool rl0 = false, rl1 = false;
  if (reg_rows) {
    if (ri0 < m) {
      ra0 = rp[ri0];
      const int d = rp[ri0 + 1] - ra0;
      rl0 = d <= kCrossLight;
      rna = rl0 ? d : 0;
      rpl0 = pl[ri0];
      rrk0 = rk[ri0];
    }
    if (ri1 < m) {
      rb0 = rp[ri1];
      const int d = rp[ri1 + 1] - rb0;
      rl1 = d <= kCrossLight;
      rnb = rl1 ? d : 0;
      rpl1 = pl[ri1];
      rrk1 = rk[ri1];
    }
  }
#pragma unroll
  for (int q = 0; q < kLctaRegIdx; ++q) {
    ria[q] = reg_rows && q < rna ? es[ra0 + q] : 0;
    rib[q] = reg_rows && q < rnb ? es[rb0 + q] : 0;
  }
  if (fast) {
    // byte offsets into buffer 0 of the interleaved vectors; slots past the
    // row read the zero slot (unpredicated loads: no per-slot predicates)
    const char* smb = reinterpret_cast<const char*>(sm);
    int oa[kLctaRegIdx], ob[kLctaRegIdx];
#pragma unroll
    for (int q = 0; q < kLctaRegIdx; ++q) {
      oa[q] = 8 * lcta_il(q < rna ? ria[q] : m);
      ob[q] = 8 * lcta_il(q < rnb ? rib[q] : m);
    }
    const int own0 = 8 * lcta_il(rl0 ? ri0 : m + 1), own1 = 8 * lcta_il(rl1 ? ri1 : m + 1);
    // one iteration reading vector B (0/1) and writing the other; true = stop
    auto step = [&](auto bsel) -> bool {
      constexpr int rd = decltype(bsel)::value * 128, wr = 128 - rd;
      double va[kLctaRegIdx], vb[kLctaRegIdx];
#pragma unroll
      for (int q = 0; q < kLctaRegIdx; ++q) {
        va[q] = *reinterpret_cast<const double*>(smb + oa[q] + rd);
        vb[q] = *reinterpret_cast<const double*>(smb + ob[q] + rd);
      }
      double ya = tree_sum<kLctaRegIdx>(va), yb = tree_sum<kLctaRegIdx>(vb);
      for (int g = kLctaRegIdx; g < rna || g < rnb; g += 4) {  // rows above kLctaRegIdx in-edges
        double wa[4], wb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          wa[q] = g + q < rna ? *reinterpret_cast<const double*>(smb + 8 * lcta_il(es[ra0 + g + q]) + rd) : 0.0;
          wb[q] = g + q < rnb ? *reinterpret_cast<const double*>(smb + 8 * lcta_il(es[rb0 + g + q]) + rd) : 0.0;
        }
        ya += tree_sum<4>(wa);
        yb += tree_sum<4>(wb);
      }
      unsigned long long lmax = 0ull;
      if (rl0) {
        rrk0 += ya;
        *reinterpret_cast<double*>(const_cast<char*>(smb) + own0 + wr) = rpl0 * ya;
        lmax = dbits(ya);
      }
      if (rl1) {
        rrk1 += yb;
        *reinterpret_cast<double*>(const_cast<char*>(smb) + own1 + wr) = rpl1 * yb;
        lmax = max(lmax, dbits(yb));
      }
      const double mx = bitsd(block_max_bits(lmax, rb2[it & 1]));
      ++it;
      if (it > cap) {
        fail = true;
        return true;
      }
      return !(mx >= tol);
    };
    for (;;) {
      if (step(std::integral_constant<int, 0>{})) break;
      if (step(std::integral_constant<int, 1>{})) break;
    }
  } else
  for (;;) {
#ifdef LR_LCTA_PROBE
    cyc_t0 = clock64();
#endif
    unsigned long long lmax = 0ull;
    if (reg_rows) {
      double ya = 0.0, yb = 0.0;
      {
        double va[kLctaRegIdx], vb[kLctaRegIdx];
#pragma unroll
        for (int q = 0; q < kLctaRegIdx; ++q) {  // (predicated: no shared-memory traffic past the row)
          va[q] = q < rna ? sc[ria[q]] : 0.0;
          vb[q] = q < rnb ? sc[rib[q]] : 0.0;
        }
        ya = tree_sum<kLctaRegIdx>(va);  // (predicated-off terms are +0.0: exact)
        yb = tree_sum<kLctaRegIdx>(vb);
      }
      double va[4], vb[4];
      for (int g = kLctaRegIdx; g < rna || g < rnb; g += 4) {  // rows above kLctaRegIdx in-edges
        int ia[4], ib[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          ia[q] = g + q < rna ? es[ra0 + g + q] : 0;
          ib[q] = g + q < rnb ? es[rb0 + g + q] : 0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          va[q] = g + q < rna ? sc[ia[q]] : 0.0;
          vb[q] = g + q < rnb ? sc[ib[q]] : 0.0;
        }
        ya += tree_sum<4>(va);
        yb += tree_sum<4>(vb);
      }
      if (rl0) {
        rrk0 += ya;
        sn[ri0] = rpl0 * ya;
        lmax = max(lmax, dbits(ya));
      }
      if (rl1) {
        rrk1 += yb;
        sn[ri1] = rpl1 * yb;
        lmax = max(lmax, dbits(yb));
      }
    } else
    // Two rows per thread in flight together; each row's in-edges in groups
    // of four (indices, then values, then the adds in order), so a row costs
    // two shared-memory round trips per group instead of two per edge.
    for (int i0 = threadIdx.x; i0 < m; i0 += 2 * kThreads) {
      const int i1 = i0 + kThreads;
      const bool has1 = i1 < m;
      const int a0 = rp[i0], a1 = rp[i0 + 1];
      const int b0 = has1 ? rp[i1] : 0, b1 = has1 ? rp[i1 + 1] : 0;
      const bool light0 = a1 - a0 <= kCrossLight, light1 = has1 && b1 - b0 <= kCrossLight;
      const int na = light0 ? a1 - a0 : 0, nb = light1 ? b1 - b0 : 0;
      double ya = 0.0, yb = 0.0;
      for (int g = 0; g < na || g < nb; g += 4) {
        int ia[4], ib[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          ia[q] = g + q < na ? es[a0 + g + q] : 0;
          ib[q] = g + q < nb ? es[b0 + g + q] : 0;
        }
        double va[4], vb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          va[q] = sc[ia[q]];
          vb[q] = sc[ib[q]];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (g + q < na) ya += va[q];
          if (g + q < nb) yb += vb[q];
        }
      }
      if (light0) {
        rk[i0] += ya;
        sn[i0] = pl[i0] * ya;
        lmax = max(lmax, dbits(ya));
      }
      if (light1) {
        rk[i1] += yb;
        sn[i1] = pl[i1] * yb;
        lmax = max(lmax, dbits(yb));
      }
    }
    if (t.pad) {  // the unit has rows above kCrossLight
      for (int base = warp * 32; base < m; base += kWarpsPer * 32) {
        const int i = base + lane;
        const int d = i < m ? rp[i + 1] - rp[i] : 0;
        unsigned mask = __ballot_sync(0xffffffffu, d > kCrossLight);
        while (mask) {
          const int src = __ffs(mask) - 1;
          mask &= mask - 1;
          const int row = base + src;
          double y = 0.0;
          for (int e = rp[row] + lane; e < rp[row + 1]; e += 32) y += sc[es[e]];
          y = warp_sum(y);
          if (lane == 0) {
            rk[row] += y;
            sn[row] = pl[row] * y;
            lmax = max(lmax, dbits(y));
          }
        }
      }
    }
#ifdef LR_LCTA_PROBE
    cyc_t1 = clock64();
    cyc_rows += cyc_t1 - cyc_t0;
#endif
    const double mx = bitsd(block_max_bits(lmax, rb2[it & 1]));
#ifdef LR_LCTA_PROBE
    cyc_max += clock64() - cyc_t1;
#endif
    double* tmp = sc;
    sc = sn;
    sn = tmp;
    ++it;
    if (it > cap) {
      fail = true;
      break;
    }
    if (!(mx >= tol)) break;
  }
  if (reg_rows) {  // register accumulators of the light rows back to shared memory
    if (rl0) rk[ri0] = rrk0;
    if (rl1) rk[ri1] = rrk1;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < m; i += kThreads) rank[rb + i] = rk[i];
#ifdef LR_LCTA_PROBE
  if (threadIdx.x == 0)
    printf("lcta unit %d m %d ne %d pad %d it %lld rows %lld max %lld cycles/iter\n", t.unit, m, ne, t.pad, it,
           cyc_rows / it, cyc_max / it);
#endif
  if (threadIdx.x == 0) {
    unit_iters[t.unit] = it;
    atomicAdd(reinterpret_cast<unsigned long long*>(&st->total_iterations), static_cast<unsigned long long>(it));
    atomicAdd(reinterpret_cast<unsigned long long*>(&st->iterative_edge_work),
              static_cast<unsigned long long>(it * t.edges));
    if (fail) atomicOr(&st->err, kErrNoConv);
  }
}

// Fallback when the unit does not fit lcta_solve_staged: in-edges read from global memory.
// The whole power series of one SccLarge unit in one CTA (solve_large_scc,
// solvers.cpp:128-162): pushed vectors in shared memory, one thread per row in
// the reference's order (bit-exact), a warp for rows above kCrossLight.
__device__ void lcta_solve(const DeviceLayout& L, const SccTask& t, int maxrows, const SolveParams* __restrict__ p,
                           const double* __restrict__ pf, double* rank, long long* unit_iters, DevStatus* st,
                           double* sm, double (*red)[32]) {
  const int rb = t.row_begin, m = t.row_end - t.row_begin;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sc = sm;
  double* sn = sm + maxrows;
  double* pl = sm + 2 * maxrows;
  const double tol = p->tol;
  const long long cap = p->cap;
  for (int i = threadIdx.x; i < m; i += kThreads) {
    pl[i] = pf[rb + i];
    sc[i] = pl[i] * rank[rb + i];
  }
  __syncthreads();
  long long it = 0;
  bool fail = false;
  for (;;) {
    double lmax = 0.0;
    for (int i = threadIdx.x; i < m; i += kThreads) {
      const int row = rb + i;
      const long long e0 = L.iptr[row], e1 = L.iptr[row + 1];
      if (e1 - e0 > kCrossLight) continue;
      double y = 0.0;
      for (long long e = e0; e < e1; ++e) y += sc[__ldg(L.isrc + e) - rb];
      rank[row] += y;
      sn[i] = pl[i] * y;
      lmax = fmax(lmax, y);
    }
    if (t.pad) {  // the unit has rows above kCrossLight
      for (int base = warp * 32; base < m; base += kWarpsPer * 32) {
        const int i = base + lane;
        long long d = 0;
        if (i < m) d = L.iptr[rb + i + 1] - L.iptr[rb + i];
        unsigned mask = __ballot_sync(0xffffffffu, d > kCrossLight);
        while (mask) {
          const int src = __ffs(mask) - 1;
          mask &= mask - 1;
          const int row = rb + base + src;
          double y = 0.0;
          for (long long e = L.iptr[row] + lane; e < L.iptr[row + 1]; e += 32) y += sc[__ldg(L.isrc + e) - rb];
          y = warp_sum(y);
          if (lane == 0) {
            rank[row] += y;
            sn[base + src] = pl[base + src] * y;
            lmax = fmax(lmax, y);
          }
        }
      }
    }
    const double mx = block_max(lmax, red[it & 1]);
    double* tmp = sc;
    sc = sn;
    sn = tmp;
    ++it;
    if (it > cap) {
      fail = true;
      break;
    }
    if (!(mx >= tol)) break;
  }
  if (threadIdx.x == 0) {
    unit_iters[t.unit] = it;
    atomicAdd(reinterpret_cast<unsigned long long*>(&st->total_iterations), static_cast<unsigned long long>(it));
    atomicAdd(reinterpret_cast<unsigned long long*>(&st->iterative_edge_work),
              static_cast<unsigned long long>(it * t.edges));
    if (fail) atomicOr(&st->err, kErrNoConv);
  }
}

// ------------------------------------------------------------- dispatcher
// Optional per-CTA timing of k_level (LR_LEVEL_PROF): task type, start, end (ns).
long long* g_level_prof = nullptr;  // host copy of the per-CTA timing buffer (LR_LEVEL_PROF)

__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifndef LR_LEVEL_MINB
#define LR_LEVEL_MINB 1
#endif
// HEAVY = the level has SccSmall or CTA power-series tasks.  Levels of row
// gathers and CAC sweeps only (most CTAs of wide levels: config 3's last level
// has 34k) run the light instantiation: no dense-solve registers, 64 per thread,
// four CTAs per SM instead of two for these latency-bound tasks.
template <bool HEAVY>
#ifndef LR_LIGHT_MINB
#define LR_LIGHT_MINB 4
#endif
__global__ void __launch_bounds__(kThreads, HEAVY ? LR_LEVEL_MINB : LR_LIGHT_MINB)
    k_level(DeviceLayout L, const LevelTask* __restrict__ tasks, const CacTask* __restrict__ cacs,
            const int* __restrict__ depth_ptr, const SccTask* __restrict__ smalls, const SccTask* __restrict__ lctas,
            int small_ld, int lcta_rows, const double* __restrict__ w, const SolveParams* __restrict__ p,
            const double* __restrict__ pf, double* rank, double* s0, long long* unit_iters, DevStatus* st,
            size_t smem_bytes, long long* prof, double* xpart) {
  extern __shared__ double sm[];
  __shared__ double red[2][32];
  const LevelTask t = tasks[blockIdx.x];
  const double c = p->c;
  const long long t_start = prof ? global_ns() : 0;
  switch (t.type) {
    case kTaskRows:
      if (smem_bytes >= kRowTaskSmem)
        cross_rows_tiled(L, t.a, t.b, w, c, pf, rank, s0, sm + (threadIdx.x >> 5) * kTileNnzCross);
      else
        cross_rows(L, t.a, t.b, w, c, pf, rank, s0, threadIdx.x, kThreads);
      break;
    case kTaskRowsPart:  // heavy instantiation only, launched with kRowTaskSmem or more
      if constexpr (HEAVY)
        cross_rows_tiled<kTaskRowsPart>(L, t.a, t.b, w, c, pf, rank, s0, sm + (threadIdx.x >> 5) * kTileNnzCross,
                                        t.split, xpart);
      break;
    case kTaskRowsFin:
      if constexpr (HEAVY)
        cross_rows_tiled<kTaskRowsFin>(L, t.a, t.b, w, c, pf, rank, s0, sm + (threadIdx.x >> 5) * kTileNnzCross,
                                       t.split, xpart);
      break;
    case kTaskCacWarps: {
      const int ci = t.a + static_cast<int>(threadIdx.x >> 5);
      if (ci >= t.b) break;
      const CacTask ct = cacs[ci];
      const int lane = threadIdx.x & 31;
      cross_rows(L, ct.row_begin, ct.row_end, w, c, pf, rank, s0, lane, 32);
      __threadfence_block();
      __syncwarp();
      const size_t per_warp = (smem_bytes / kWarpsPer) & ~static_cast<size_t>(15);
      if (cac_stage_bytes(ct.row_end - ct.row_begin, L.iptr[ct.row_end] - L.iptr[ct.row_begin]) <= per_warp)
        cac_sweep_staged<false>(L, ct, depth_ptr, c, rank, lane, 32,
                                reinterpret_cast<unsigned char*>(sm) + per_warp * (threadIdx.x >> 5));
      else
        cac_sweep<false>(L, ct, depth_ptr, c, rank, lane, 32);
      break;
    }
    case kTaskCacBlock: {
      const CacTask ct = cacs[t.a];
      cross_rows_cta(L, ct.row_begin, ct.row_end, w, c, pf, rank, s0, sm, smem_bytes, kWarpsPer);
      __syncthreads();
      if (cac_stage_bytes(ct.row_end - ct.row_begin, L.iptr[ct.row_end] - L.iptr[ct.row_begin]) <= smem_bytes)
        cac_sweep_staged<true>(L, ct, depth_ptr, c, rank, threadIdx.x, kThreads, sm);
      else
        cac_sweep<true>(L, ct, depth_ptr, c, rank, threadIdx.x, kThreads);
      break;
    }
    case kTaskSmall: {
      if constexpr (HEAVY) {
        const SccTask sct = smalls[t.a];
        cross_rows_cta(L, sct.row_begin, sct.row_end, w, c, pf, rank, s0, sm, smem_bytes, kWarpsPer);
        __syncthreads();
        small_dispatch(L, sct, small_ld, c, pf, rank, sm, red[0], st);
      }
      break;
    }
    case kTaskLcta: {
      if constexpr (HEAVY) {
        const SccTask lt = lctas[t.a];
        cross_rows_cta(L, lt.row_begin, lt.row_end, w, c, pf, rank, s0, sm, smem_bytes, kWarpsPer);
        __syncthreads();
        if (lcta_stage_bytes(lcta_rows, L.iptr[lt.row_end] - L.iptr[lt.row_begin]) <= smem_bytes)
          lcta_solve_staged(L, lt, lcta_rows, p, pf, rank, unit_iters, st, sm, red);
        else
          lcta_solve(L, lt, lcta_rows, p, pf, rank, unit_iters, st, sm, red);
      }
      break;
    }
    default:
      break;
  }
  if (prof) {
    __syncthreads();
    if (threadIdx.x == 0) {
      prof[3 * blockIdx.x] = t.type;
      prof[3 * blockIdx.x + 1] = t_start;
      prof[3 * blockIdx.x + 2] = global_ns();
    }
  }
}

// Large CACs (kCacMidMaxRows < rows <= kCacBlockMaxRows): one 1024-thread CTA
// per CAC gathers its rows' start weights and runs the depth sweep, on a side
// stream concurrently with the level's k_level (config 4: one such CAC per
// level, ~20 us, formerly serialised after k_level).
constexpr int kBigThreads = 1024;


__global__ void __launch_bounds__(kBigThreads)
    k_cac_big(DeviceLayout L, const CacTask* __restrict__ cacs, const int* __restrict__ depth_ptr,
              const double* __restrict__ w, const SolveParams* __restrict__ p, const double* __restrict__ pf,
              double* rank, double* s0, double* pv, size_t smem_bytes, long long* prof) {
  extern __shared__ double sm[];
  const CacTask ct = cacs[blockIdx.x];
  const long long t_start = prof ? global_ns() : 0;

  // the CAC's own start weights (rows above kCrossSplit cross in-edges were
  // done by k_pull_heavy before the level), so the launch runs concurrently
  // with the level's k_level on a side stream
  if (!ct.pregathered) {
    cross_rows_cta(L, ct.row_begin, ct.row_end, w, p->c, pf, rank, s0, sm, smem_bytes, kBigThreads / 32);
    __syncthreads();
  }
  const int m = ct.row_end - ct.row_begin;
  const long long ne = L.iptr[ct.row_end] - L.iptr[ct.row_begin];
  if (cac_stage_bytes(m, ne) <= smem_bytes)
    cac_sweep_staged<true>(L, ct, depth_ptr, p->c, rank, threadIdx.x, kBigThreads, sm);
  else if (pv != nullptr && m < 65536 && cac_compact_bytes(m, ne) <= smem_bytes)
    cac_sweep_compact(L, ct, depth_ptr, p->c, rank, pv, sm);
  else
    cac_sweep<true>(L, ct, depth_ptr, p->c, rank, threadIdx.x, kBigThreads);
  if (prof) {
    __syncthreads();
    if (threadIdx.x == 0) {
      prof[3 * blockIdx.x] = 0;
      prof[3 * blockIdx.x + 1] = t_start;
      prof[3 * blockIdx.x + 2] = global_ns();
    }
  }
}

}  // namespace

void launch_cac_big(const DeviceLayout& L, const CacTask* cacs, int n, const int* depth_ptr, const double* w,
                    const SolveParams* p, const double* pf, double* rank, double* s0, double* pv, size_t smem,
                    cudaStream_t s, long long* task_times) {
  if (n == 0) return;
  // highest launch priority (kept by graph capture): its 1024-thread CTAs need a
  // whole SM and must be placed before the level's k_level CTAs fill them
  static const int prio = [] {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    return hi;
  }();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(n));
  cfg.blockDim = dim3(kBigThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = prio;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_cac_big, L, cacs, depth_ptr, w, p, pf, rank, s0, pv, smem, task_times);
}

size_t cac_stage_need(long long rows, long long edges) { return cac_stage_bytes(rows, edges); }
size_t cac_compact_need(long long rows, long long edges) { return cac_compact_bytes(rows, edges); }

cudaError_t configure_level_kernel() {
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes a{};
  e = cudaFuncGetAttributes(&a, k_level<true>);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_level<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           optin - static_cast<int>(a.sharedSizeBytes));
  if (e != cudaSuccess) return e;
  e = cudaFuncGetAttributes(&a, k_level<false>);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_level<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           optin - static_cast<int>(a.sharedSizeBytes));
  if (e != cudaSuccess) return e;
  e = cudaFuncGetAttributes(&a, k_cac_big);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_cac_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin - static_cast<int>(a.sharedSizeBytes));
}

cudaError_t set_level_prof(long long* buf) {
  g_level_prof = buf;
  return cudaSuccess;
}

void launch_level(const DeviceLayout& L, const LevelTask* tasks, int ntasks, const CacTask* cacs, const int* depth_ptr,
                  const SccTask* smalls, const SccTask* lctas, int small_ld, int lcta_rows, size_t smem,
                  const double* w, const SolveParams* p, const double* pf, double* rank, double* s0,
                  long long* unit_iters, DevStatus* st, bool heavy, cudaStream_t s, bool profile, double* xpart,
                  long long* task_times) {
  if (ntasks == 0) return;
  // per-CTA (type, start ns, end ns): the level profile (one launch per level
  // owns that buffer) or the per-unit timing buffer of this launch's tasks
  long long* prof = task_times ? task_times : profile ? g_level_prof : nullptr;
  if (heavy)
    k_level<true><<<ntasks, kThreads, smem, s>>>(L, tasks, cacs, depth_ptr, smalls, lctas, small_ld, lcta_rows, w, p,
                                                 pf, rank, s0, unit_iters, st, smem, prof, xpart);
  else
    k_level<false><<<ntasks, kThreads, smem, s>>>(L, tasks, cacs, depth_ptr, smalls, lctas, small_ld, lcta_rows, w, p,
                                                  pf, rank, s0, unit_iters, st, smem, prof, xpart);
}

}  // namespace lrk
