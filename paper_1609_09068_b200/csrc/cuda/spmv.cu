// K4b: the grid-wide power-series iteration of the large SCC units
// (solve_large_scc, proj/src/solvers.cpp:146-160) -- the dominant kernel.
//
// Pull SpMV y_i = sum_{j in in(i)} s_j over the unit's in-edge CSR, fused with
// rank_i += y_i, s'_i = pf_i * y_i and the max-norm stop test.  Work is cut on
// the host into warp tasks of <= kTileNnz in-edges:
//   tile      rows [row_begin,row_end) whole, <= kTileRows rows
//   long row  one row with kTileNnz < in-degree <= kSegNnz
//   segment   kSegNnz in-edges of a heavier row; partials combined in segment
//             order by whichever segment finishes last
// One persistent CTA per SM of kHeadWarps warps.  Random 8-byte gathers cost
// one L1 wavefront per distinct 128-byte line, which bounds this kernel; the
// layout orders a unit's rows by in-unit out-degree, so the most-gathered
// pushed values sit at the head of the unit, and each CTA stages that head
// (up to ~19.6k doubles) in shared memory once per launch: gathers that land
// there cost a bank access instead of a line.  Every warp walks its own
// strided slice of the task list and never waits on another warp: a tile
// issues its 8 index loads per lane, its row offsets and epilogue operands,
// then the 8 gathers, stages them in a warp-private buffer and reduces rows.
// Rows up to kLongRow in-edges are summed by one lane in the reference's own
// order (bit-exact with the CPU push scatter); longer rows use a butterfly.
#include <cuda_runtime.h>

#include "devutil.cuh"
#include "kernels.cuh"

namespace lrk {
namespace {

using namespace dev;

constexpr int kHeadWarps = 32;                  // warps per persistent CTA
constexpr int kHeadThreads = kHeadWarps * 32;
constexpr int kPerLane = kTileNnz / 32;
constexpr int kLongRow = 32;
constexpr int kStageBytes = kHeadWarps * (kTileNnz * 8 + (kTileRows + 1) * 4 + 12);

__global__ void k_grid_reset(GridUnitState* gs, int ngu, DevStatus* st) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ngu) {
    gs[i].max_bits = 0ull;
    gs[i].iterations = 0;
    gs[i].done = 0;
  }
  if (i == 0) {
    st->active = ngu;
    st->ctas_done = 0;
  }
}

// Run by the last CTA of a launch: closes the iteration of every unit of the
// level -- stop when max|inc| < tol (solvers.cpp:160), fail past the cap (:159).
__device__ void finish_iteration(GridUnitState* gs, int gu0, int ngu, const SolveParams* p, long long* unit_iters,
                                 DevStatus* st) {
  for (int i = gu0; i < gu0 + ngu; ++i) {
    GridUnitState* u = gs + i;
    if (u->done) continue;
    const double mx = bitsd(atomicAdd(&u->max_bits, 0ull));
    const int it = u->iterations + 1;
    u->iterations = it;
    u->max_bits = 0ull;
    bool stop = false;
    if (it > p->cap) {
      atomicOr(&st->err, kErrNoConv);
      stop = true;
    } else if (!(mx >= p->tol)) {
      stop = true;
    }
    if (stop) {
      u->done = 1;
      unit_iters[u->unit] = it;
      atomicAdd(reinterpret_cast<unsigned long long*>(&st->total_iterations), static_cast<unsigned long long>(it));
      atomicAdd(reinterpret_cast<unsigned long long*>(&st->iterative_edge_work),
                static_cast<unsigned long long>(static_cast<long long>(it) * u->edges));
      atomicSub(&st->active, 1);
    }
  }
  st->ctas_done = 0;
}

__device__ __forceinline__ void epilogue(int row, double y, double rk, double pfr, double* rank, double* s_out,
                                         double& lmax) {
  rank[row] = rk + y;
  s_out[row] = pfr * y;
  lmax = fmax(lmax, y);
}

// s_in[i] through the shared head when i lies in [head_base, head_base + nhead).
__device__ __forceinline__ double gather(const double* __restrict__ s_in, const double* head, int head_base,
                                         int nhead, int i) {
  const unsigned h = static_cast<unsigned>(i - head_base);
  return h < static_cast<unsigned>(nhead) ? head[h] : __ldg(s_in + i);
}

__global__ void __launch_bounds__(kHeadThreads, 1)
    k_grid_iter(DeviceLayout L, const SpmvBlock* __restrict__ tasks, int ntasks, int gu0, int ngu, GridUnitState* gs,
                const HeavyRow* __restrict__ heavy, double* heavy_part, int* heavy_cnt,
                const SolveParams* __restrict__ p, const double* __restrict__ pf, double* __restrict__ rank,
                const double* __restrict__ s_in, double* __restrict__ s_out, long long* unit_iters, DevStatus* st,
                int head_base, int nhead) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* head = reinterpret_cast<double*>(smem);
  double* vals = head + nhead;                                          // [kHeadWarps][kTileNnz]
  int* rp = reinterpret_cast<int*>(vals + kHeadWarps * kTileNnz);       // [kHeadWarps][kTileRows + 1]
  int* wunit = rp + kHeadWarps * (kTileRows + 1);
  double* wmax = reinterpret_cast<double*>(wunit + kHeadWarps + (kHeadWarps & 1));
  __shared__ int last_cta;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* v = vals + warp * kTileNnz;
  int* wr = rp + warp * (kTileRows + 1);

  // stage the hot head of the pushed vector (read-only during this launch)
  if (nhead > 0) {
    const double2* src = reinterpret_cast<const double2*>(s_in + head_base);
    double2* dst = reinterpret_cast<double2*>(head);
    const bool aligned = (head_base & 1) == 0;
    for (int i = threadIdx.x; i < (nhead >> 1); i += blockDim.x)
      dst[i] = aligned ? __ldg(src + i) : make_double2(__ldg(s_in + head_base + 2 * i), __ldg(s_in + head_base + 2 * i + 1));
    if ((nhead & 1) && threadIdx.x == 0) head[nhead - 1] = __ldg(s_in + head_base + nhead - 1);
    __syncthreads();
  }

  int cur_unit = -1;
  double lmax = 0.0;
  const int stride = gridDim.x * kHeadWarps;
  for (int t = blockIdx.x * kHeadWarps + warp; t < ntasks; t += stride) {
    const SpmvBlock b = tasks[t];
    if (b.gunit != cur_unit) {
      if (cur_unit >= 0) {
        const double m = warp_max(lmax);
        if (lane == 0 && m > 0.0) atomicMax(&gs[cur_unit].max_bits, dbits(m));
      }
      cur_unit = b.gunit;
      lmax = 0.0;
    }
    if (gs[b.gunit].done) continue;
    if (b.heavy < 0 && b.nnz <= kTileNnz) {
      int idx[kPerLane];
#pragma unroll
      for (int k = 0; k < kPerLane; ++k) {
        const int e = lane + 32 * k;
        idx[k] = e < b.nnz ? __ldg(L.isrc + b.nnz_begin + e) : -1;
      }
      const int nr = b.row_end - b.row_begin;
      for (int i = lane; i <= nr; i += 32) wr[i] = static_cast<int>(__ldg(L.iptr + b.row_begin + i) - b.nnz_begin);
      double rk[kTileRows / 32], pfr[kTileRows / 32];
#pragma unroll
      for (int j = 0; j < kTileRows / 32; ++j) {
        const int r = lane + 32 * j;
        rk[j] = r < nr ? rank[b.row_begin + r] : 0.0;
        pfr[j] = r < nr ? __ldg(pf + b.row_begin + r) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < kPerLane; ++k)
        if (idx[k] >= 0) v[lane + 32 * k] = gather(s_in, head, head_base, nhead, idx[k]);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < kTileRows / 32; ++j) {
        const int r = lane + 32 * j;
        if (r >= nr) continue;
        const int lo = wr[r], hi = wr[r + 1];
        if (hi - lo > kLongRow) continue;
        double y = 0.0;
        for (int k = lo; k < hi; ++k) y += v[k];
        epilogue(b.row_begin + r, y, rk[j], pfr[j], rank, s_out, lmax);
      }
      for (int r = 0; r < nr; ++r) {
        const int lo = wr[r], hi = wr[r + 1];
        if (hi - lo <= kLongRow) continue;
        double y = 0.0;
        for (int k = lo + lane; k < hi; k += 32) y += v[k];
        y = warp_sum(y);
        const int row = b.row_begin + r;
        if (lane == 0) epilogue(row, y, rank[row], pf[row], rank, s_out, lmax);
      }
      __syncwarp();
    } else {
      double part = 0.0;
      for (int base = 0; base < b.nnz; base += kTileNnz) {
        int idx[kPerLane];
#pragma unroll
        for (int k = 0; k < kPerLane; ++k) {
          const int e = base + lane + 32 * k;
          idx[k] = e < b.nnz ? __ldg(L.isrc + b.nnz_begin + e) : -1;
        }
#pragma unroll
        for (int k = 0; k < kPerLane; ++k)
          if (idx[k] >= 0) part += gather(s_in, head, head_base, nhead, idx[k]);
      }
      part = warp_sum(part);
      if (b.heavy < 0) {
        if (lane == 0) epilogue(b.row_begin, part, rank[b.row_begin], pf[b.row_begin], rank, s_out, lmax);
      } else if (lane == 0) {
        const HeavyRow h = heavy[b.heavy];
        heavy_part[h.part_begin + b.seg] = part;
        __threadfence();
        if (atomicAdd(heavy_cnt + b.heavy, 1) == h.nseg - 1) {
          __threadfence();
          double y = 0.0;
          for (int k = 0; k < h.nseg; ++k) y += __ldcg(heavy_part + h.part_begin + k);
          heavy_cnt[b.heavy] = 0;
          epilogue(h.row, y, rank[h.row], pf[h.row], rank, s_out, lmax);
        }
      }
    }
  }
  const double m = warp_max(lmax);
  if (lane == 0) {
    wunit[warp] = cur_unit;
    wmax[warp] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < kHeadWarps; ++w) {
      if (wunit[w] < 0 || !(wmax[w] > 0.0)) continue;
      double mm = wmax[w];
      while (w + 1 < kHeadWarps && wunit[w + 1] == wunit[w]) mm = fmax(mm, wmax[++w]);
      atomicMax(&gs[wunit[w]].max_bits, dbits(mm));
    }
    __threadfence();
    last_cta = atomicAdd(&st->ctas_done, 1) == static_cast<int>(gridDim.x) - 1;
  }
  __syncthreads();
  if (last_cta && threadIdx.x == 0) {
    __threadfence();
    finish_iteration(gs, gu0, ngu, p, unit_iters, st);
  }
}

int blocks_for(long long n, int threads) { return static_cast<int>((n + threads - 1) / threads); }

int optin_smem() {
  static int v = 0;
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes a{};
    cudaFuncGetAttributes(&a, k_grid_iter);
    v -= static_cast<int>(a.sharedSizeBytes);
    cudaFuncSetAttribute(k_grid_iter, cudaFuncAttributeMaxDynamicSharedMemorySize, v);
  }
  return v;
}

}  // namespace

int grid_iter_ctas() {
  static int ctas = 0;
  if (ctas == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&ctas, cudaDevAttrMultiProcessorCount, dev);
  }
  return ctas;
}

int grid_head_capacity() { return (optin_smem() - kStageBytes - 64) / 8 & ~1; }

void launch_grid_reset(GridUnitState* gs, int ngu, DevStatus* st, cudaStream_t s) {
  k_grid_reset<<<blocks_for(ngu > 0 ? ngu : 1, 128), 128, 0, s>>>(gs, ngu, st);
}

void launch_grid_iter(const DeviceLayout& L, const SpmvBlock* tasks, int ntasks, int gu0, int ngu, GridUnitState* gs,
                      const HeavyRow* heavy, double* heavy_part, int* heavy_cnt, const SolveParams* p, const double* pf,
                      double* rank, const double* s_in, double* s_out, long long* unit_iters, DevStatus* st,
                      int head_base, int nhead, cudaStream_t s) {
  if (ntasks == 0) return;
  const int cap = grid_head_capacity();
  if (nhead > cap) nhead = cap;
  if (nhead < 0) nhead = 0;
  const size_t bytes = static_cast<size_t>(nhead) * 8 + kStageBytes + 16;
  k_grid_iter<<<grid_iter_ctas(), kHeadThreads, bytes, s>>>(L, tasks, ntasks, gu0, ngu, gs, heavy, heavy_part,
                                                            heavy_cnt, p, pf, rank, s_in, s_out, unit_iters, st,
                                                            head_base, nhead);
}

}  // namespace lrk
