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
// Persistent CTAs; every warp walks its own strided slice of the task list and
// never waits on another warp.  The kernel is bound by random 8-byte gathers
// (one L1 wavefront and one L2 sector per distinct line), so it keeps as many
// of them in flight as it can and keeps the gathered vector resident in L2:
//   * a tile issues its 8 index loads per lane, its row offsets and epilogue
//     operands, then all 8 gathers back to back (clamped addresses instead of
//     branches, so nothing serialises them), then stages them in a
//     warp-private shared buffer and reduces rows;
//   * streamed data (indices, row pointers, rank, pf) is loaded with an L2
//     evict-first policy and without L1 allocation, the gathered pushed vector
//     s with evict-last, and the next pushed vector s' is stored evict-last --
//     the row order (descending in-unit out-degree) packs the most-gathered
//     entries together, so they stay in L2 across iterations.
// Rows up to kLongRow in-edges are summed by one lane in the reference's own
// order (bit-exact with the CPU push scatter); longer rows use a butterfly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "devutil.cuh"
#include "kernels.cuh"

namespace lrk {
namespace {

using namespace dev;

constexpr int kWarps = kSpmvThreads / 32;
constexpr int kPerLane = kTileNnz / 32;
constexpr int kLongRow = 32;
constexpr int kHeadRows = 8192;  // shared-memory head entries of K4b (see launch_grid_iter)
constexpr int kHeadRowsSeg = 16384;  // ... of K4c

// L2 priority of the streamed operands (indices, row offsets, rank, pf):
// evict-first when they cannot stay resident across iterations, evict-last when
// the whole level's working set fits in L2 (then nothing is re-read from HBM)
__device__ __forceinline__ std::uint64_t policy_stream(int keep) {
  std::uint64_t p;
  if (keep == 2)
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else if (keep == 1)
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  else
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// evict-last for the hot head [base, base + primary) of a pushed vector,
// evict-first for the rest of the unit [base + primary, base + total)
__device__ __forceinline__ std::uint64_t policy_hot_head(const double* base, unsigned primary, unsigned total) {
  std::uint64_t p;
  asm("createpolicy.range.global.L2::evict_last.L2::evict_first.b64 %0, [%1], %2, %3;"
      : "=l"(p)
      : "l"(base), "r"(primary), "r"(total));
  return p;
}
// streamed, read-only: no L1 allocation, first out of L2
__device__ __forceinline__ int ld_stream(const int* p, std::uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ long long ld_stream(const long long* p, std::uint64_t pol) {
  long long v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_stream(const double* p, std::uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
// The gathered pushed vector.  Its hottest columns -- the first rows of the
// degree-ordered unit, the target of most in-edges -- are copied into shared
// memory at the start of each launch; a gather reads shared memory when its
// column is in that head and global memory (no L1 allocation) otherwise.  Both
// loads are issued predicated and selected afterwards (no branch, so all of a
// chunk's gathers stay in flight together).
__device__ __forceinline__ double ld_keep(const double* p, std::uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_gather(const double* gp, unsigned sh, unsigned in_head, std::uint64_t pol) {
  double a = 0.0, b = 0.0;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared.f64 %0, [%1];\n\t}"
      : "+d"(a)
      : "r"(sh), "r"(in_head));
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.eq.u32 q, %2, 0;\n\t@q ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], "
      "%3;\n\t}"
      : "+d"(b)
      : "l"(gp), "r"(in_head), "l"(pol));
  return in_head ? a : b;
}
__device__ __forceinline__ void st_keep(double* p, double v, std::uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

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
    st->last_max = 0.0;
    st->prev_max = 0.0;
    st->next_task = 0;
  }
}

// Run by the last CTA of a launch: closes the iteration of every unit of the
// level -- stop when max|inc| < tol (solvers.cpp:160), fail past the cap (:159).
// `maxbuf` (multi-GPU): the all-reduced maxima of the row shards, else this
// launch's own max.
__device__ void finish_iteration(GridUnitState* gs, int gu0, int ngu, const SolveParams* p, long long* unit_iters,
                                 DevStatus* st, const double* maxbuf = nullptr) {
  double level_max = 0.0;
  for (int i = gu0; i < gu0 + ngu; ++i) {
    GridUnitState* u = gs + i;
    if (u->done) continue;
    const double mx = maxbuf ? maxbuf[i] : bitsd(atomicAdd(&u->max_bits, 0ull));
    level_max = fmax(level_max, mx);
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
  st->prev_max = st->last_max;
  st->last_max = level_max;
  st->ctas_done = 0;
}

__global__ void __launch_bounds__(kSpmvThreads)
    k_grid_iter(DeviceLayout L, const SpmvBlock* __restrict__ tasks, int ntasks, int gu0, int ngu, GridUnitState* gs,
                const HeavyRow* __restrict__ heavy, double* heavy_part, int* heavy_cnt,
                const SolveParams* __restrict__ p, const double* __restrict__ pf, double* __restrict__ rank,
                const double* __restrict__ s_in, double* __restrict__ s_out, long long* unit_iters, DevStatus* st,
                int hot_begin, unsigned hot_bytes, unsigned unit_bytes, int nhead, int keep_stream, double* maxbuf, int hold) {
  extern __shared__ double dyn[];  // [kWarps][kTileNnz] staging, then the head
  double* head = dyn + kWarps * kTileNnz;
  __shared__ int wunit[kWarps];
  __shared__ double wmax[kWarps];
  __shared__ int last_cta;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* v = dyn + warp * kTileNnz;
  const std::uint64_t stream = policy_stream(keep_stream);
  const std::uint64_t keep = policy_hot_head(s_in + hot_begin, hot_bytes, unit_bytes);
  const std::uint64_t keep_out = policy_hot_head(s_out + hot_begin, hot_bytes, unit_bytes);
  int cur_unit = -1;
  double lmax = 0.0;
  const int stride = gridDim.x * kWarps;
  // this launch's copy of the hot head of s_in (read-only for the launch)
  for (int i = threadIdx.x; i < nhead; i += kSpmvThreads) head[i] = ld_keep(s_in + hot_begin + i, keep);
  const unsigned head_sh = static_cast<unsigned>(__cvta_generic_to_shared(head));
  __syncthreads();

  // Software pipeline over 256-edge chunks (a tile is one chunk, long rows and
  // segments up to four): the index loads of chunk i+1 are issued together
  // with the gathers and row operands of chunk i, so each chunk costs one
  // memory round trip instead of two.
  auto seek = [&](int& tt, SpmvBlock& bb) {  // first task at or after tt whose unit still iterates
    while (tt < ntasks) {
      bb = tasks[tt];
      if (!gs[bb.gunit].done) return;
      tt += stride;
    }
  };
  auto load_idx = [&](const SpmvBlock& bb, int cc, int* out) {
    const int* src = L.isrc + bb.nnz_begin + static_cast<long long>(cc) * kTileNnz;
    const int left = bb.nnz - cc * kTileNnz;
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {
      const int e = lane + 32 * k;
      out[k] = ld_stream(src + (e < left ? e : 0), stream);
    }
  };
  int t = blockIdx.x * kWarps + warp, c = 0;
  SpmvBlock b{};
  seek(t, b);
  int idx[kPerLane];
  if (t < ntasks) load_idx(b, 0, idx);
  double part = 0.0;  // running sum of a multi-chunk task
  while (t < ntasks) {
    if (b.gunit != cur_unit) {
      if (cur_unit >= 0) {
        const double m = warp_max(lmax);
        if (lane == 0 && m > 0.0) atomicMax(&gs[cur_unit].max_bits, dbits(m));
      }
      cur_unit = b.gunit;
      lmax = 0.0;
    }
    const bool tile = b.heavy < 0 && b.nnz <= kTileNnz;
    const int left = b.nnz - c * kTileNnz;
    // 1. this chunk's gathers
    double g[kPerLane];
#pragma unroll
    for (int k = 0; k < kPerLane; ++k)
    {
      const unsigned off = static_cast<unsigned>(idx[k] - hot_begin);
      const unsigned in = off < static_cast<unsigned>(nhead);
      g[k] = ld_gather(s_in + idx[k], head_sh + (in ? off : 0u) * 8u, in, keep);
    }
    // 2. this tile's row operands, in flight with the gathers
    const int nr = tile ? b.row_end - b.row_begin : 0;
    int lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;
    double rk0 = 0.0, rk1 = 0.0, pf0 = 0.0, pf1 = 0.0;
    if (tile) {
      const long long* ip = L.iptr + b.row_begin;
      const int r0 = lane < nr ? lane : nr - 1, r1 = lane + 32 < nr ? lane + 32 : nr - 1;
      lo0 = static_cast<int>(ld_stream(ip + r0, stream) - b.nnz_begin);
      hi0 = static_cast<int>(ld_stream(ip + r0 + 1, stream) - b.nnz_begin);
      lo1 = static_cast<int>(ld_stream(ip + r1, stream) - b.nnz_begin);
      hi1 = static_cast<int>(ld_stream(ip + r1 + 1, stream) - b.nnz_begin);
      rk0 = ld_stream(rank + b.row_begin + r0, stream);
      pf0 = ld_stream(pf + b.row_begin + r0, stream);
      rk1 = ld_stream(rank + b.row_begin + r1, stream);
      pf1 = ld_stream(pf + b.row_begin + r1, stream);
    }
    // 3. the next chunk's indices
    int tn = t, cn = c + 1;
    SpmvBlock bn = b;
    if (cn * kTileNnz >= b.nnz) {
      tn = t + stride;
      cn = 0;
      seek(tn, bn);
    }
    int idx_n[kPerLane];
    if (tn < ntasks) load_idx(bn, cn, idx_n);
    // 4. consume this chunk
    if (tile) {
#pragma unroll
      for (int k = 0; k < kPerLane; ++k)
        if (lane + 32 * k < b.nnz) v[lane + 32 * k] = g[k];
      __syncwarp();
      const bool live0 = lane < nr, live1 = lane + 32 < nr;
      if (live0 && hi0 - lo0 <= kLongRow) {
        double y = 0.0;
        for (int k = lo0; k < hi0; ++k) y += v[k];
        rank[b.row_begin + lane] = rk0 + y;
        st_keep(s_out + b.row_begin + lane, pf0 * y, keep_out);
        lmax = fmax(lmax, y);
      }
      if (live1 && hi1 - lo1 <= kLongRow) {
        double y = 0.0;
        for (int k = lo1; k < hi1; ++k) y += v[k];
        rank[b.row_begin + lane + 32] = rk1 + y;
        st_keep(s_out + b.row_begin + lane + 32, pf1 * y, keep_out);
        lmax = fmax(lmax, y);
      }
      // rows longer than kLongRow: one warp butterfly each
      for (int half = 0; half < 2; ++half) {
        const bool is_long = half == 0 ? (live0 && hi0 - lo0 > kLongRow) : (live1 && hi1 - lo1 > kLongRow);
        unsigned mask = __ballot_sync(0xffffffffu, is_long);
        while (mask) {
          const int src = __ffs(mask) - 1;
          mask &= mask - 1;
          const int lo = __shfl_sync(0xffffffffu, half == 0 ? lo0 : lo1, src);
          const int hi = __shfl_sync(0xffffffffu, half == 0 ? hi0 : hi1, src);
          const double rk = __shfl_sync(0xffffffffu, half == 0 ? rk0 : rk1, src);
          const double pr = __shfl_sync(0xffffffffu, half == 0 ? pf0 : pf1, src);
          double y = 0.0;
          for (int k = lo + lane; k < hi; k += 32) y += v[k];
          y = warp_sum(y);
          if (lane == 0) {
            const int row = b.row_begin + src + 32 * half;
            rank[row] = rk + y;
            st_keep(s_out + row, pr * y, keep_out);
            lmax = fmax(lmax, y);
          }
        }
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int k = 0; k < kPerLane; ++k)
        if (lane + 32 * k < left) part += g[k];
      if (left <= kTileNnz) {  // last chunk of a long row or segment
        const double sum = warp_sum(part);
        part = 0.0;
        int row = -1;
        double y = sum;
        if (b.heavy < 0) {
          row = b.row_begin;
        } else if (lane == 0) {
          const HeavyRow h = heavy[b.heavy];
          heavy_part[h.part_begin + b.seg] = sum;
          __threadfence();
          if (atomicAdd(heavy_cnt + b.heavy, 1) == h.nseg - 1) {
            __threadfence();
            y = 0.0;
            for (int k = 0; k < h.nseg; ++k) y += __ldcg(heavy_part + h.part_begin + k);
            heavy_cnt[b.heavy] = 0;
            row = h.row;
          }
        }
        if (lane == 0 && row >= 0) {
          rank[row] += y;
          st_keep(s_out + row, pf[row] * y, keep_out);
          lmax = fmax(lmax, y);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) idx[k] = idx_n[k];
    t = tn;
    c = cn;
    b = bn;
  }
  const double m = warp_max(lmax);
  if (lane == 0) {
    wunit[warp] = cur_unit;
    wmax[warp] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < kWarps; ++w) {
      if (wunit[w] < 0 || !(wmax[w] > 0.0)) continue;
      double mm = wmax[w];
      while (w + 1 < kWarps && wunit[w + 1] == wunit[w]) mm = fmax(mm, wmax[++w]);
      atomicMax(&gs[wunit[w]].max_bits, dbits(mm));
    }
    __threadfence();
    last_cta = atomicAdd(&st->ctas_done, 1) == static_cast<int>(gridDim.x) - 1;
  }
  __syncthreads();
  if (last_cta && threadIdx.x == 0) {
    __threadfence();
    if (hold) {  // an earlier chunk of a chunked (multi-GPU) iteration: maxima keep accumulating
      st->ctas_done = 0;
    } else if (maxbuf) {  // row-sharded: publish the shard max, decide after the all-reduce
      for (int i = gu0; i < gu0 + ngu; ++i) {
        maxbuf[i] = bitsd(atomicAdd(&gs[i].max_bits, 0ull));
        gs[i].max_bits = 0ull;
      }
      st->ctas_done = 0;
    } else {
      finish_iteration(gs, gu0, ngu, p, unit_iters, st);
    }
  }
}

// K4c: the same iteration with every lane owning 8 CONSECUTIVE in-edges of a
// chunk (one 256-bit index load), rows reduced by a segmented warp scan instead
// of a shared-memory staging buffer -- fewer instructions per edge, no serial
// per-lane row loops, and the shared memory the staging took goes to the head.
//   chunk  in-edges [cb, cb + n), n <= kChunkNnz, inside the aligned window
//          [A, A + 256), A = cb & ~7: lane l owns slots 8l .. 8l + 7
//   tile   rows [row_begin, row_end) whole (one chunk); row r starts at slot
//          iptr[r] - A.  Row-start flags (8 bitmap words per warp in shared
//          memory) give each lane its rows; a lane sums its own complete rows,
//          rows crossing lanes are combined by an inclusive segmented scan.
//   long row / heavy-row segment: one row, up to four chunks, warp sum.
// Summation order differs from the reference's sequential push (rows agree to
// ~1e-16 relative; the stop test and iteration counts are unaffected).
__device__ __forceinline__ void ld_idx8(const int* p, std::uint64_t pol, int* o) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]), "=r"(o[7])
               : "l"(p), "l"(pol));
}

__device__ __forceinline__ SpmvBlock from_lanes(int v) {
  SpmvBlock r;
  const unsigned lo = static_cast<unsigned>(__shfl_sync(0xffffffffu, v, 0));
  const int hi = __shfl_sync(0xffffffffu, v, 1);
  r.nnz_begin = static_cast<long long>(lo) | (static_cast<long long>(hi) << 32);
  r.nnz = __shfl_sync(0xffffffffu, v, 2);
  r.row_begin = __shfl_sync(0xffffffffu, v, 3);
  r.row_end = __shfl_sync(0xffffffffu, v, 4);
  r.gunit = __shfl_sync(0xffffffffu, v, 5);
  r.heavy = __shfl_sync(0xffffffffu, v, 6);
  r.seg = __shfl_sync(0xffffffffu, v, 7);
  return r;
}

__device__ __forceinline__ unsigned ld_meta(const unsigned short* p, std::uint64_t pol) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
  return v;
}

// A chunk in flight: its task, its gathers and (tiles) its row operands.
#ifndef LR_SEG_PIPE
#define LR_SEG_PIPE 1
#endif
struct SegStage {
  SpmvBlock b;
  int t, c;
  unsigned mt;  // tile lane metadata
  double g[8];
  double rk0, rk1, pf0, pf1;
};

__global__ void __launch_bounds__(kSegThreads, 1)
    k_spmv_seg(DeviceLayout L, const SpmvBlock* __restrict__ tasks, const unsigned short* __restrict__ meta,
               int ntasks, int gu0, int ngu, GridUnitState* gs, const HeavyRow* __restrict__ heavy,
               double* heavy_part, int* heavy_cnt, const SolveParams* __restrict__ p, const double* __restrict__ pf,
               double* __restrict__ rank, const double* __restrict__ s_in, double* __restrict__ s_out,
               long long* unit_iters, DevStatus* st, int hot_begin, unsigned hot_bytes, unsigned unit_bytes,
               int nhead, int keep_stream, double* maxbuf, int hold) {
  constexpr int kW = kSegThreads / 32;
  extern __shared__ double dyn[];  // [kW][kTileRows] row totals, then the head
  double* head = dyn + kW * kTileRows;
  __shared__ int wunit[kW];
  __shared__ double wmax[kW];
  __shared__ unsigned char sdone[kMaxSharedUnits];
  __shared__ int last_cta;
  __shared__ int cta_next;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) cta_next = 0;
  const std::uint64_t stream = policy_stream(keep_stream);
  const std::uint64_t keep = policy_hot_head(s_in + hot_begin, hot_bytes, unit_bytes);
  const std::uint64_t keep_out = policy_hot_head(s_out + hot_begin, hot_bytes, unit_bytes);
  int live = 0;
  for (int i = threadIdx.x; i < ngu; i += kSegThreads) {
    const int d = gs[gu0 + i].done;
    live |= !d;
    if (i < kMaxSharedUnits) sdone[i] = d ? 1 : 0;
  }
  live = __syncthreads_or(live);  // launches past convergence exit at once
  if (live)
    for (int i = threadIdx.x; i < nhead; i += kSegThreads) head[i] = ld_keep(s_in + hot_begin + i, keep);
  __syncthreads();
  // generic addresses of column j: glob_base + 8 j, or (head) head_base + 8 j
  const long long glob_base = reinterpret_cast<long long>(s_in);
  const long long head_base = reinterpret_cast<long long>(head) - 8ll * hot_begin;
  auto unit_done = [&](int gu) {
    const int i = gu - gu0;
    return i < kMaxSharedUnits ? sdone[i] != 0 : gs[gu].done != 0;
  };
  // CTA b owns tasks b, b + grid, b + 2 grid, ... (the whole grid sweeps the
  // rows in order); its warps claim them one at a time from a shared counter,
  // so no warp idles at the end of a launch while another of its CTA still
  // has a static share left.
  auto grab = [&]() {
    int v = ntasks;
    if (lane == 0 && live) {
      const long long k = atomicAdd(&cta_next, 1);
      const long long tt = blockIdx.x + k * gridDim.x;
      v = tt < ntasks ? static_cast<int>(tt) : ntasks;
    }
    return __shfl_sync(0xffffffffu, v, 0);
  };
  // The descriptor of the next task to claim is loaded one task ahead (lane
  // i < 8 holds its int i); its unit's done flag is checked on arrival.
  int tq = grab();
  int bq = 0;
  if (tq < ntasks && lane < 8) bq = __ldg(reinterpret_cast<const int*>(tasks + tq) + lane);
  auto next_task = [&](int& tt, SpmvBlock& bb) {
    for (;;) {
      tt = tq;
      if (tt >= ntasks) return;
      bb = from_lanes(bq);
      tq = grab();
      if (tq < ntasks && lane < 8) bq = __ldg(reinterpret_cast<const int*>(tasks + tq) + lane);
      if (!unit_done(bb.gunit)) return;
    }
  };
  // the chunk after (tt, bb, cc): the next chunk of the same task or the
  // first chunk of the next task
  auto advance = [&](int& tt, SpmvBlock& bb, int& cc) {
    if ((cc + 1) * kChunkNnz < bb.nnz) {
      ++cc;
    } else {
      cc = 0;
      next_task(tt, bb);
    }
  };
  // a chunk's 8 index slots and, for a tile, its lane metadata (row-start
  // flags of my 8 slots | rows starting before them << 8)
  auto load_chunk = [&](int tt, const SpmvBlock& bb, int cc, int* out, unsigned& mt) {
    const long long cb = bb.nnz_begin + static_cast<long long>(cc) * kChunkNnz;
    ld_idx8(L.isrc + (cb & ~7ll) + 8 * lane, stream, out);
    mt = bb.heavy < 0 && bb.nnz <= kChunkNnz ? ld_meta(meta + static_cast<long long>(tt) * 32 + lane, stream) : 0u;
  };
  // issue a chunk's gathers (valid slots [q0, q1) of its window) and its tile's row operands
  auto issue = [&](SegStage& S, const int* idx) {
    const int left = S.b.nnz - S.c * kChunkNnz;
    const int q0 = static_cast<int>((S.b.nnz_begin + static_cast<long long>(S.c) * kChunkNnz) & 7ll);
    const int q1 = q0 + (left < kChunkNnz ? left : kChunkNnz);
    const int lo = min(max(q0 - 8 * lane, 0), 8), hi = min(max(q1 - 8 * lane, 0), 8);
    const unsigned vm = (0xffu >> (8 - hi)) & (0xffu << lo) & 0xffu;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      // one generic load: the shared-memory head or the global pushed vector
      const unsigned off = static_cast<unsigned>(idx[k] - hot_begin);
      LR_DCHECK(!(vm & (1u << k)) || (idx[k] >= 0 && idx[k] < L.n));
      const long long base = off < static_cast<unsigned>(nhead) ? head_base : glob_base;
      const double* src = reinterpret_cast<const double*>(base + (static_cast<long long>(idx[k]) << 3));
      double v = 0.0;
      asm volatile(
          "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %3;\n\t}"
          : "+d"(v)
          : "l"(src), "r"(vm & (1u << k)), "l"(keep));
      S.g[k] = v;
    }
    const bool tile = S.b.heavy < 0 && S.b.nnz <= kChunkNnz;
    const int nr = tile ? S.b.row_end - S.b.row_begin : 0;
    S.rk0 = S.rk1 = S.pf0 = S.pf1 = 0.0;
    if (lane < nr) {
      S.rk0 = ld_stream(rank + S.b.row_begin + lane, stream);
      S.pf0 = ld_stream(pf + S.b.row_begin + lane, stream);
    }
    if (lane + 32 < nr) {
      S.rk1 = ld_stream(rank + S.b.row_begin + lane + 32, stream);
      S.pf1 = ld_stream(pf + S.b.row_begin + lane + 32, stream);
    }
  };
  int cur_unit = -1;
  double lmax = 0.0;
  double part = 0.0;  // running sum of a multi-chunk task
  // consume a chunk whose gathers have been issued
  auto consume = [&](const SegStage& S) {
    const SpmvBlock& b = S.b;
    if (b.gunit != cur_unit) {
      if (cur_unit >= 0) {
        const double m = warp_max(lmax);
        if (lane == 0 && m > 0.0) atomicMax(&gs[cur_unit].max_bits, dbits(m));
      }
      cur_unit = b.gunit;
      lmax = 0.0;
    }
    if (b.heavy < 0 && b.nnz <= kChunkNnz) {
      const int nr = b.row_end - b.row_begin;
      double* ysh = dyn + warp * kTileRows;
      const unsigned mine = S.mt & 0xffu;             // row starts among my 8 slots
      const int before = static_cast<int>(S.mt >> 8);  // rows starting before my first slot
      // my complete rows go straight to ysh; `pre` continues a row begun in an
      // earlier lane, `run` ends as the part of a row continued by later lanes
      double pre = 0.0, run = 0.0;
      int o = before - 1;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if ((mine >> k) & 1u) {
          if (o >= before) ysh[o] = run;
          else pre = run;
          ++o;
          run = 0.0;
        }
        run += S.g[k];
      }
      // inclusive segmented scan over lanes; segments start at lanes with a row start
      const unsigned fl = __ballot_sync(0xffffffffu, mine != 0u);
      const unsigned upto = fl & (0xffffffffu >> (31 - lane));
      const int seg0 = upto ? 31 - __clz(upto) : 0;
      double v = run;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double vu = __shfl_up_sync(0xffffffffu, v, d);
        if (lane - d >= seg0) v += vu;
      }
      const double prev = __shfl_up_sync(0xffffffffu, v, 1);
      if (mine && before > 0) ysh[before - 1] = (lane > 0 ? prev : 0.0) + pre;
      const int last_lane = (static_cast<int>((b.nnz_begin & 7ll)) + b.nnz - 1) >> 3;
      if (b.nnz > 0 && lane == last_lane) ysh[nr - 1] = v;
      __syncwarp();
      if (lane < nr) {
        const double y = b.nnz > 0 ? ysh[lane] : 0.0;  // nnz = 0: a run of rows without in-edges
        rank[b.row_begin + lane] = S.rk0 + y;
        st_keep(s_out + b.row_begin + lane, S.pf0 * y, keep_out);
        lmax = fmax(lmax, y);
      }
      if (lane + 32 < nr) {
        const double y = b.nnz > 0 ? ysh[lane + 32] : 0.0;
        rank[b.row_begin + lane + 32] = S.rk1 + y;
        st_keep(s_out + b.row_begin + lane + 32, S.pf1 * y, keep_out);
        lmax = fmax(lmax, y);
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) part += S.g[k];
      if (b.nnz - S.c * kChunkNnz <= kChunkNnz) {  // last chunk of a long row or segment
        const double sum = warp_sum(part);
        part = 0.0;
        int row = -1;
        double y = sum;
        if (b.heavy < 0) {
          row = b.row_begin;
        } else if (lane == 0) {
          const HeavyRow h = heavy[b.heavy];
          heavy_part[h.part_begin + b.seg] = sum;
          __threadfence();
          if (atomicAdd(heavy_cnt + b.heavy, 1) == h.nseg - 1) {
            __threadfence();
            y = 0.0;
            for (int k = 0; k < h.nseg; ++k) y += __ldcg(heavy_part + h.part_begin + k);
            heavy_cnt[b.heavy] = 0;
            row = h.row;
          }
        }
        if (lane == 0 && row >= 0) {
          rank[row] += y;
          st_keep(s_out + row, pf[row] * y, keep_out);
          lmax = fmax(lmax, y);
        }
      }
    }
  };
  // Two chunks in flight per warp: while chunk A is reduced, the gathers of
  // chunk B are outstanding and the indices of the chunk after B are loading.
  SegStage A, B;
  int idx[8];
  A.c = 0;
  next_task(A.t, A.b);
  if (A.t < ntasks) {
    load_chunk(A.t, A.b, 0, idx, A.mt);
    issue(A, idx);
    B.t = A.t;
    B.b = A.b;
    B.c = A.c;
    advance(B.t, B.b, B.c);
    if (B.t < ntasks) load_chunk(B.t, B.b, B.c, idx, B.mt);
  }
  while (A.t < ntasks) {
    int tn = B.t, cn = B.c;
    SpmvBlock bn = B.b;
    unsigned mtn = 0u;
#if LR_SEG_PIPE == 1
    consume(A);  // one chunk in flight: B's gathers wait for A's reduction
#endif
    if (B.t < ntasks) {
      issue(B, idx);
      advance(tn, bn, cn);
      if (tn < ntasks) load_chunk(tn, bn, cn, idx, mtn);
    }
#if LR_SEG_PIPE != 1
    consume(A);
#endif
    A = B;
    B.t = tn;
    B.b = bn;
    B.c = cn;
    B.mt = mtn;
  }
  const double m = warp_max(lmax);
  if (lane == 0) {
    wunit[warp] = cur_unit;
    wmax[warp] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < kW; ++w) {
      if (wunit[w] < 0 || !(wmax[w] > 0.0)) continue;
      double mm = wmax[w];
      while (w + 1 < kW && wunit[w + 1] == wunit[w]) mm = fmax(mm, wmax[++w]);
      atomicMax(&gs[wunit[w]].max_bits, dbits(mm));
    }
    __threadfence();
    last_cta = atomicAdd(&st->ctas_done, 1) == static_cast<int>(gridDim.x) - 1;
  }
  __syncthreads();
  if (last_cta && threadIdx.x == 0) {
    __threadfence();
    if (hold) {  // an earlier chunk of a chunked (multi-GPU) iteration: maxima keep accumulating
      st->ctas_done = 0;
    } else if (maxbuf) {  // row-sharded: publish the shard max, decide after the all-reduce
      for (int i = gu0; i < gu0 + ngu; ++i) {
        maxbuf[i] = bitsd(atomicAdd(&gs[i].max_bits, 0ull));
        gs[i].max_bits = 0ull;
      }
      st->ctas_done = 0;
    } else {
      finish_iteration(gs, gu0, ngu, p, unit_iters, st);
    }
  }
}

// K5: one power-series iteration of a large grid unit by dest-row blocks
// (DESIGN.md §4.1 "K5").  A CTA claims parts (a contiguous range of one
// block's in-edges, sorted by source) from a global counter; its warps walk the
// part 256 slots at a time, lane l taking slots l, l+32, ... (stored lane-major,
// so its 8 sources and 8 dest rows are two vector loads), so each
// gather instruction reads 32 CONSECUTIVE sources of the sorted list: where the
// sources are dense (the high-degree rows that carry most in-edges) they share
// 128-byte lines and one L2 request serves many in-edges -- the pull SpMV's
// one-request-per-in-edge ceiling does not apply.  Rows accumulate in shared
// memory (y[BR]; unused slots carry dst = BR and are skipped; the entries are
// placed so that a half-warp's dest rows lie on distinct bank pairs, blk.cu); a
// whole block is finished by
// its CTA (rank += y, s' = pf y, max), a split block's parts add their rows into
// yacc and the last one to arrive finishes them.  Summation order depends on
// the atomics' arrival order (rows agree to ~1e-16; iteration counts asserted).
// a lane's 8 slots of a chunk (slot lane + 32 k, stored at lane * 8 + k): 8
// sources with one 256-bit load, 8 dest rows with one 128-bit load
__device__ __forceinline__ void ld_blk_idx(const unsigned* es, const unsigned short* ed, int lane,
                                           std::uint64_t pol, unsigned (&j)[8], unsigned (&d)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=r"(j[0]), "=r"(j[1]), "=r"(j[2]), "=r"(j[3]), "=r"(j[4]), "=r"(j[5]), "=r"(j[6]), "=r"(j[7])
               : "l"(es + lane * 8), "l"(pol));
  unsigned q[4];
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3])
               : "l"(ed + lane * 8), "l"(pol));
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    d[2 * m] = q[m] & 0xffffu;
    d[2 * m + 1] = q[m] >> 16;
  }
}
template <int GATHER_L1>
__device__ __forceinline__ double ld_blk_gather(const double* p, std::uint64_t pol) {
  double v;
  if (GATHER_L1)
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

template <int GATHER_L1, int PIPE>
__global__ void __launch_bounds__(kBlkThreads, 1)
    k_spmv_blk(BlkUnitDev B, int gu, GridUnitState* gs, const SolveParams* __restrict__ p,
               const double* __restrict__ pf, double* __restrict__ rank, const double* __restrict__ s_in,
               double* __restrict__ s_out, long long* unit_iters, DevStatus* st, int hot_begin, unsigned hot_bytes,
               unsigned unit_bytes, double* maxbuf, int hold) {
  constexpr int kW = kBlkThreads / 32;
  extern __shared__ double y[];  // [BR + 1]
  __shared__ int s_part;
  __shared__ int s_last;
  __shared__ double wmax[kW];
  if (gs[gu].done) return;  // launches past convergence exit at once
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::uint64_t stream = policy_stream(0);
  const std::uint64_t keep = policy_hot_head(s_in + hot_begin, hot_bytes, unit_bytes);
  const std::uint64_t keep_out = policy_hot_head(s_out + hot_begin, hot_bytes, unit_bytes);
  const double* sb = s_in + B.u0;
  const unsigned ubr = static_cast<unsigned>(B.BR);
  double lmax = 0.0;
  auto finish_row = [&](int r, double v) {
    const long long g = static_cast<long long>(B.row0) + r;
    // rank and pf pass through once per iteration: first out of L2
    double rk;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(rk) : "l"(rank + g), "l"(stream));
    st_keep(rank + g, rk + v, stream);
    st_keep(s_out + g, ld_stream(pf + g, stream) * v, keep_out);
    lmax = fmax(lmax, v);
  };
  for (;;) {
    if (threadIdx.x == 0) s_part = atomicAdd(&st->next_task, 1);
    for (int i = threadIdx.x; i <= B.BR; i += kBlkThreads) y[i] = 0.0;
    __syncthreads();
    const int pi = s_part;
    if (pi >= B.nparts) break;
    const BlkPart P = B.parts[pi];
    const unsigned* es = B.esrc + P.e0;
    const unsigned short* ed = B.edst + P.e0;
    if (PIPE) {
      // the next chunk's indices load while this chunk's gathers are in flight
      int c = warp * kBlkChunk;
      unsigned j[8], d[8];
      if (c < P.n) ld_blk_idx(es + c, ed + c, lane, stream, j, d);
      for (; c < P.n; c += kW * kBlkChunk) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          LR_DCHECK(j[k] < static_cast<unsigned>(B.UR) && d[k] <= static_cast<unsigned>(B.BR));
          v[k] = ld_blk_gather<GATHER_L1>(sb + j[k], keep);
        }
        const int cn = c + kW * kBlkChunk;
        unsigned jn[8], dn[8];
        if (cn < P.n) ld_blk_idx(es + cn, ed + cn, lane, stream, jn, dn);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (d[k] != ubr) atomicAdd(y + d[k], v[k]);  // dummies (unused slots) add nothing
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          j[k] = jn[k];
          d[k] = dn[k];
        }
      }
    } else {
      for (int c = warp * kBlkChunk; c < P.n; c += kW * kBlkChunk) {
        unsigned j[8], d[8];
        ld_blk_idx(es + c, ed + c, lane, stream, j, d);
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          LR_DCHECK(j[k] < static_cast<unsigned>(B.UR) && d[k] <= static_cast<unsigned>(B.BR));
          v[k] = ld_blk_gather<GATHER_L1>(sb + j[k], keep);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (d[k] != ubr) atomicAdd(y + d[k], v[k]);  // dummies (unused slots) add nothing
      }
    }
    __syncthreads();
    const int r0 = P.blk * B.BR, nr = min(B.BR, B.R - r0);
    if (P.slot < 0) {
      for (int i = threadIdx.x; i < nr; i += kBlkThreads) finish_row(r0 + i, y[i]);
    } else {
      double* ya = B.yacc + static_cast<size_t>(P.slot) * B.BR;
      for (int i = threadIdx.x; i < nr; i += kBlkThreads) atomicAdd(ya + i, y[i]);
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) s_last = atomicAdd(B.bcnt + P.slot, 1) == P.nsplit - 1;
      __syncthreads();
      if (s_last) {
        __threadfence();
        for (int i = threadIdx.x; i < nr; i += kBlkThreads) {
          const double v = __ldcg(ya + i);
          ya[i] = 0.0;
          finish_row(r0 + i, v);
        }
        if (threadIdx.x == 0) B.bcnt[P.slot] = 0;
      }
    }
    __syncthreads();  // y is zeroed for the next part
  }
  const double m = warp_max(lmax);
  if (lane == 0) wmax[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = 0.0;
    for (int w = 0; w < kW; ++w) mm = fmax(mm, wmax[w]);
    if (mm > 0.0) atomicMax(&gs[gu].max_bits, dbits(mm));
    __threadfence();
    s_last = atomicAdd(&st->ctas_done, 1) == static_cast<int>(gridDim.x) - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    st->next_task = 0;
    if (hold) {  // an earlier chunk of a chunked (multi-GPU) iteration: the maximum keeps accumulating
      st->ctas_done = 0;
    } else if (maxbuf) {  // row-sharded: publish the shard max, decide after the all-reduce
      maxbuf[gu] = bitsd(atomicAdd(&gs[gu].max_bits, 0ull));
      gs[gu].max_bits = 0ull;
      st->ctas_done = 0;
    } else {
      finish_iteration(gs, gu, 1, p, unit_iters, st);
    }
  }
}

__global__ void k_grid_finish(GridUnitState* gs, int gu0, int ngu, const SolveParams* p, long long* unit_iters,
                              DevStatus* st, const double* maxbuf) {
  if (threadIdx.x == 0 && blockIdx.x == 0) finish_iteration(gs, gu0, ngu, p, unit_iters, st, maxbuf);
}

// a shard whose last chunk of an iteration is empty: publish what the earlier
// chunks accumulated
__global__ void k_grid_publish(GridUnitState* gs, double* maxbuf, int gu0, int ngu) {
  const int i = gu0 + static_cast<int>(threadIdx.x);
  if (i < gu0 + ngu) {
    maxbuf[i] = bitsd(gs[i].max_bits);
    gs[i].max_bits = 0ull;
  }
}

__global__ void k_grid_zero_max(double* maxbuf, int gu0, int ngu) {
  const int i = threadIdx.x;
  if (i < ngu) maxbuf[gu0 + i] = 0.0;
}

int blocks_for(long long n, int threads) { return static_cast<int>((n + threads - 1) / threads); }

}  // namespace

// K4c (k_spmv_seg) unless LR_SPMV=tile selects the staged-tile kernel K4b.
bool spmv_seg() {
  static const bool seg = [] {
    const char* e = std::getenv("LR_SPMV");
    return !(e && std::string(e) == "tile");
  }();
  return seg;
}

// Dynamic shared memory: at most as many head entries as fit next to the
// per-warp buffers (staging for K4b, row totals for K4c).
static int head_capacity() {
  static int cap = -1;
  if (cap < 0) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes a{};
    const int per_warp = spmv_seg() ? (kSegThreads / 32) * kTileRows : kWarps * kTileNnz;
    if (spmv_seg()) {
      cudaFuncGetAttributes(&a, k_spmv_seg);
    } else {
      cudaFuncGetAttributes(&a, k_grid_iter);
    }
    cap = ((optin - static_cast<int>(a.sharedSizeBytes)) / 8 - per_warp) / 32 * 32;
    const int bytes = (cap + per_warp) * 8;
    if (spmv_seg())
      cudaFuncSetAttribute(k_spmv_seg, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    else
      cudaFuncSetAttribute(k_grid_iter, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  }
  return cap;
}

int grid_iter_ctas() {
  static int ctas = 0;
  if (ctas == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_warp = spmv_seg() ? (kSegThreads / 32) * kTileRows : kWarps * kTileNnz;
    const size_t bytes = static_cast<size_t>(head_capacity() + per_warp) * 8;
    if (spmv_seg())
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_seg, kSegThreads, bytes);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_grid_iter, kSpmvThreads, bytes);
    ctas = sms * (per_sm > 0 ? per_sm : 1);
  }
  return ctas;
}

void launch_grid_reset(GridUnitState* gs, int ngu, DevStatus* st, cudaStream_t s) {
  k_grid_reset<<<blocks_for(ngu > 0 ? ngu : 1, 128), 128, 0, s>>>(gs, ngu, st);
}

void launch_grid_iter(const DeviceLayout& L, const SpmvBlock* tasks, const unsigned short* meta, int ntasks, int gu0,
                      int ngu, GridUnitState* gs, const HeavyRow* heavy, double* heavy_part, int* heavy_cnt, const SolveParams* p, const double* pf,
                      double* rank, const double* s_in, double* s_out, long long* unit_iters, DevStatus* st,
                      int hot_begin, long long hot_rows, long long unit_rows, int keep_stream, double* maxbuf,
                      cudaStream_t s, int hold) {
  if (ntasks == 0) {  // no rows of the level's units in this launch
    if (maxbuf && !hold) k_grid_publish<<<1, 1024, 0, s>>>(gs, maxbuf, gu0, ngu);
    return;
  }
  const unsigned hot_bytes = static_cast<unsigned>(hot_rows * 8), unit_bytes = static_cast<unsigned>(unit_rows * 8);
  const int want = blocks_for(ntasks, spmv_seg() ? kSegThreads / 32 : kWarps);
  const int grid = want < grid_iter_ctas() ? want : grid_iter_ctas();
  // Head size: measured optimum 4-12k entries at configs 2 and 5 for K4b.
  // Larger heads lose: the fill costs microseconds per launch, and the L1 left
  // over holds the in-flight misses of the cold gathers.  LR_SPMV_HEAD
  // overrides (0 disables the head).
  // K4c: 16k entries while the pushed vector is L2-resident (configs 2, 3),
  // 8k for vectors far beyond L2 (config 5: the cold gathers need the L1)
  int want_head = spmv_seg() ? (unit_rows * 8 <= (48ll << 20) ? kHeadRowsSeg : kHeadRows) : kHeadRows;
  if (const char* e = std::getenv("LR_SPMV_HEAD")) want_head = std::max(0, std::atoi(e));
  const int nhead = static_cast<int>(std::min<long long>({head_capacity(), want_head, unit_rows}));
  if (spmv_seg()) {
    k_spmv_seg<<<grid, kSegThreads, static_cast<size_t>(nhead + (kSegThreads / 32) * kTileRows) * 8, s>>>(
        L, tasks, meta, ntasks, gu0, ngu, gs, heavy, heavy_part, heavy_cnt, p, pf, rank, s_in, s_out, unit_iters, st,
        hot_begin, hot_bytes, unit_bytes, nhead, keep_stream, maxbuf, hold);
  } else {
    k_grid_iter<<<grid, kSpmvThreads, static_cast<size_t>(nhead + kWarps * kTileNnz) * 8, s>>>(
        L, tasks, ntasks, gu0, ngu, gs, heavy, heavy_part, heavy_cnt, p, pf, rank, s_in, s_out, unit_iters, st,
        hot_begin, hot_bytes, unit_bytes, nhead, keep_stream, maxbuf, hold);
  }
}

// K5 launch: one persistent CTA per SM (y takes BR + 1 doubles of shared memory).
// The gathers allocate in L1 (LR_BLK_L1=0: not): with the bank balance an entry
// moved to a neighbouring row finds its line already fetched by that row
// (5,110 -> 5,189 GB/s at config 5; before the balance it measured slightly
// slower, 3,924 vs 3,952); LR_BLK_PIPE=0 drops the index prefetch.
void launch_spmv_blk(const BlkUnitDev& B, int gu, GridUnitState* gs, const SolveParams* p, const double* pf,
                     double* rank, const double* s_in, double* s_out, long long* unit_iters, DevStatus* st,
                     int hot_begin, long long hot_rows, long long unit_rows, cudaStream_t s, double* maxbuf, int hold) {
  const char* e_l1 = std::getenv("LR_BLK_L1");
  const bool l1 = !(e_l1 && std::atoi(e_l1) == 0);
  const char* e_pipe = std::getenv("LR_BLK_PIPE");
  const bool pipe = !(e_pipe && std::atoi(e_pipe) == 0);
  static int sms = 0;
  static size_t smem_set = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t smem = static_cast<size_t>(B.BR + 1) * sizeof(double);
  if (smem > smem_set) {  // opt in to the block's y (static shared memory comes on top)
    cudaFuncSetAttribute(k_spmv_blk<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(k_spmv_blk<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(k_spmv_blk<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(k_spmv_blk<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    smem_set = smem;
  }
  const int grid = std::max(1, std::min(sms, B.nparts));
  const unsigned hot_bytes = static_cast<unsigned>(hot_rows * 8), unit_bytes = static_cast<unsigned>(unit_rows * 8);
  auto kern = l1 ? (pipe ? k_spmv_blk<1, 1> : k_spmv_blk<1, 0>) : (pipe ? k_spmv_blk<0, 1> : k_spmv_blk<0, 0>);
  kern<<<grid, kBlkThreads, smem, s>>>(B, gu, gs, p, pf, rank, s_in, s_out, unit_iters, st, hot_begin, hot_bytes,
                                       unit_bytes, maxbuf, hold);
}

void launch_grid_zero_max(double* maxbuf, int gu0, int ngu, cudaStream_t s) {
  k_grid_zero_max<<<1, 1024, 0, s>>>(maxbuf, gu0, ngu);
}

void launch_grid_finish(GridUnitState* gs, int gu0, int ngu, const SolveParams* p, long long* unit_iters,
                        DevStatus* st, const double* maxbuf, cudaStream_t s) {
  k_grid_finish<<<1, 32, 0, s>>>(gs, gu0, ngu, p, unit_iters, st, maxbuf);
}

}  // namespace lrk
