// Device-side build of K5's dest-blocked layout (kernels.cuh BlkUnitDev) from
// the unit's in-edge CSR already on the device (one-time setup at upload):
//   1. k_blk_keys + CUB radix sort: every in-edge keyed by (dest block, source),
//      the in-block dest row as payload.  Rows are in unit order, so block b's
//      in-edges occupy the same CSR range before and after the sort.
//   2. k_blk_pack: each block's sorted run into its slots (rows of 32 slots, one
//      empty row per `slack` rows, padded to whole chunks; unused slots = dummies).
//   3. k_blk_banks: entries placed inside windows of `win` slots so that each
//      half-warp of K5 adds to 16 distinct shared-memory bank pairs, chunks
//      stored lane-major (k_blk_lane_major alone when the balance is off).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace lrk {
namespace {

// warp per row: key = (row block << sbits) | source row in the unit
__global__ void k_blk_keys(const long long* __restrict__ iptr, const int* __restrict__ isrc, long long e_begin, int u0,
                           int row0, int R, int BR, int sbits, unsigned long long* __restrict__ keys,
                           unsigned short* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const long long w0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long r = w0; r < R; r += nw) {
    const long long g = row0 + r;
    const long long a = iptr[g], b = iptr[g + 1];
    const unsigned long long hi = static_cast<unsigned long long>(r / BR) << sbits;
    const unsigned short d = static_cast<unsigned short>(r % BR);
    for (long long e = a + lane; e < b; e += 32) {
      keys[e - e_begin] = hi | static_cast<unsigned long long>(static_cast<unsigned>(isrc[e] - u0));
      vals[e - e_begin] = d;
    }
  }
}

// thread per padded slot: sorted run -> padded slot (the slot's block by binary
// search in pad_off; the heaviest block holds a large share of all entries, so
// the work is split by slots, not by blocks).  With slack > 0 every `slack`
// instruction rows (32 slots each) of entries are followed by one empty row of
// dummies (src 0, dst BR): free slots near every entry for k_blk_banks.
__global__ void k_blk_pack(const long long* __restrict__ iptr, long long e_begin, int row0, int R, int BR,
                           const long long* __restrict__ pad_off, int nb, unsigned long long smask,
                           const unsigned long long* __restrict__ keys, const unsigned short* __restrict__ vals,
                           unsigned* __restrict__ esrc, unsigned short* __restrict__ edst, int slack) {
  const long long total = pad_off[nb];
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int lo = 0, hi = nb;  // last block with pad_off[b] <= i (empty blocks share their successor's offset)
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pad_off[mid] <= i) lo = mid;
      else hi = mid;
    }
    const int r0 = lo * BR, r1 = min(R, r0 + BR);
    const long long s0 = iptr[row0 + r0] - e_begin, cnt = iptr[row0 + r1] - iptr[row0 + r0];
    long long j = i - pad_off[lo];  // slot in the block's run -> entry of the sorted run, or -1
    if (slack > 0) {
      const long long row = j >> 5, period = slack + 1;
      j = (row % period == slack) ? -1 : (row - row / period) * 32 + (j & 31);
    }
    if (j >= 0 && j < cnt) {
      esrc[i] = static_cast<unsigned>(keys[s0 + j] & smask);
      edst[i] = vals[s0 + j];
    } else {
      esrc[i] = 0u;
      edst[i] = static_cast<unsigned short>(BR);
    }
  }
}

// Slot i of a window (instruction row i / 32, lane i % 32; windows and chunks
// start at multiples of 256) -> its place in memory: K5 stores a chunk
// lane-major (lane * 8 + row within the chunk), so a lane's 8 slots are one
// vector load.
__device__ __forceinline__ int blk_slot_pos(int i) { return (i & ~255) | ((i & 31) << 3) | ((i >> 5) & 7); }

// Shared-memory bank balance, one CTA per window of W slots (several chunks of
// one block), the window staged in shared memory.  K5 lane l of a warp handles slots l + 32 k of a chunk; its
// atomic add to y[dst] (LDS + DADD + ATOMS.CAST.SPIN.64) hits the bank pair
// dst mod 16 (8-byte words), and a half-warp whose 16 adds use 16 distinct bank
// pairs takes the fewest shared-memory wavefronts -- the L1/shared data pipe is
// what bounds K5 (profiles/r02t_cfg5_k5_ncu.md: ~3.4 wavefronts per conflict,
// one per extra 128-byte line of a gather instruction).  Two passes:
// (1) every instruction row (32 slots = two half-warps) keeps its own entries
// where it can -- the first entry of a bank pair goes to half A, the second to
// half B, any further one is left over; (2) a left-over entry moves to the
// nearest row with a free slot in a half that does not have its bank pair yet
// (dummy slots count as free); (3) whatever remains takes the nearest free slot.
// Only the conflicting entries (~13 % for random rows) leave their row, so a
// gather instruction keeps most of its 32 adjacent sources; an in-order greedy
// placement cascades instead (an entry pushed into a neighbour pushes the
// neighbour's own entries on: measured 4,700 vs 5,050 GB/s at config 5).
// The bank pairs do not interact in pass 2: a half-warp that lacks a bank pair
// has a free slot (16 slots, at most one entry per pair until pass 3), so warp c
// places the left-overs of bank pair c on its own, in order, and an entry's lane
// inside its half-warp is the rank of its bank pair among the half's pairs --
// the layout does not depend on how the warps interleave.
constexpr int kBanksThreads = 512;  // 16 warps: one per bank pair in pass 2
template <int W>
__global__ void __launch_bounds__(kBanksThreads, 1)
    k_blk_banks(unsigned* __restrict__ esrc, unsigned short* __restrict__ edst, const long long* __restrict__ wstart,
                const int* __restrict__ wlen, long long nwin, int BR, int reach) {
  constexpr int NI = W / 32;  // instruction rows of a full window
  static_assert(NI <= kBanksThreads, "one thread per row in pass 1");
  extern __shared__ unsigned char blk_smem[];
  unsigned* s = reinterpret_cast<unsigned*>(blk_smem);  // [W] entries as packed (slot order)
  unsigned* os = s + W;                                 // [W] placed
  unsigned* occ = os + W;                               // [2 NI] bank pairs taken per half-warp (low 16 bits)
  unsigned* rownear = occ + 2 * NI;                     // [NI]
  unsigned short* d = reinterpret_cast<unsigned short*>(rownear + NI);
  unsigned short* od = d + W;
  unsigned short* half = od + W;    // half-warp an entry goes to (0xffff: pass 3 decides)
  unsigned short* left = half + W;  // pass 1 left-overs, 32 per row
  unsigned char* extra = reinterpret_cast<unsigned char*>(left + W);  // [2 NI] pass 3 entries per half-warp
  unsigned char* lcnt = extra + 2 * NI;                               // [NI]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (long long wi = blockIdx.x; wi < nwin; wi += gridDim.x) {
    unsigned* es = esrc + wstart[wi];
    unsigned short* ed = edst + wstart[wi];
    const int len = wlen[wi], ni = len / 32;
    for (int i = tid; i < len; i += kBanksThreads) {
      s[i] = es[i];
      d[i] = ed[i];
      os[i] = 0u;
      od[i] = static_cast<unsigned short>(BR);
    }
    __syncthreads();
    // pass 1: a row keeps what fits its two half-warps (thread per row)
    if (tid < ni) {
      unsigned oa = 0, ob = 0;
      int nl = 0;
      for (int l = 0; l < 32; ++l) {
        const int i = tid * 32 + l;
        if (d[i] == BR) continue;  // a dummy: its slot is free
        const unsigned bit = 1u << (d[i] & 15);
        if (!(oa & bit)) {
          oa |= bit;
          half[i] = static_cast<unsigned short>(2 * tid);
        } else if (!(ob & bit)) {
          ob |= bit;
          half[i] = static_cast<unsigned short>(2 * tid + 1);
        } else {
          left[tid * 32 + nl++] = static_cast<unsigned short>(i);
        }
      }
      occ[2 * tid] = oa;
      occ[2 * tid + 1] = ob;
      extra[2 * tid] = extra[2 * tid + 1] = 0;
      lcnt[tid] = static_cast<unsigned char>(nl);
    }
    __syncthreads();
    // pass 2 (warp c = bank pair c; lane l looks at the row at distance
    // base + l / 2, after (even l) or before (odd l): the lowest lane that fits
    // is the nearest)
    if (warp < 16) {
      const unsigned bit = 1u << warp;
      for (int r = 0; r < ni; ++r)
        for (int q = 0; q < lcnt[r]; ++q) {
          const int i = left[r * 32 + q];
          if ((d[i] & 15) != warp) continue;
          int h = -1;
          for (int base = 1; base < min(ni, reach) && h < 0; base += 16) {
            const int dist = base + (lane >> 1), in = (lane & 1) ? r - dist : r + dist;
            int mine = -1;
            if (dist < ni && in >= 0 && in < ni) {
              if (!(occ[2 * in] & bit)) mine = 2 * in;
              else if (!(occ[2 * in + 1] & bit)) mine = 2 * in + 1;
            }
            const unsigned vote = __ballot_sync(0xffffffffu, mine >= 0);
            if (vote) h = __shfl_sync(0xffffffffu, mine, __ffs(vote) - 1);
          }
          if (lane == 0) {
            if (h >= 0) atomicOr(&occ[h], bit);  // other warps set other bits of the same word
            half[i] = static_cast<unsigned short>(h >= 0 ? h : 0xffff);
          }
          __syncwarp();
        }
    }
    __syncthreads();
    // pass 3 (warp 0): entries without a conflict-free half-warp anywhere in the
    // window take the nearest free slot, in order
    if (warp == 0)
      for (int i0 = 0; i0 < len; i0 += 32) {
        unsigned todo = __ballot_sync(0xffffffffu, d[i0 + lane] != BR && half[i0 + lane] == 0xffffu);
        for (; todo; todo &= todo - 1) {
          const int i = i0 + __ffs(todo) - 1, r = i >> 5;
          int h = -1;
          for (int base = 0; base < ni && h < 0; base += 16) {
            const int dist = base + (lane >> 1), in = (lane & 1) ? r - dist : r + dist;
            int mine = -1;
            if (dist < ni && !((lane & 1) && dist == 0) && in >= 0 && in < ni) {
              if (__popc(occ[2 * in]) + extra[2 * in] < 16) mine = 2 * in;
              else if (__popc(occ[2 * in + 1]) + extra[2 * in + 1] < 16) mine = 2 * in + 1;
            }
            const unsigned vote = __ballot_sync(0xffffffffu, mine >= 0);
            if (vote) h = __shfl_sync(0xffffffffu, mine, __ffs(vote) - 1);
          }
          if (lane == 0) {  // behind the half-warp's conflict-free entries
            half[i] = static_cast<unsigned short>(h | 0x8000);
            left[i] = static_cast<unsigned short>(extra[h]++);
          }
          __syncwarp();
        }
      }
    __syncthreads();
    for (int i = tid; i < len; i += kBanksThreads)
      if (d[i] != BR) {
        const int h = half[i] & 0x7fff;
        const unsigned o = occ[h], bit = 1u << (d[i] & 15);
        // conflict-free entries by the rank of their bank pair, pass 3 entries behind them
        const int lane_in_half = (half[i] & 0x8000) ? __popc(o) + left[i] : __popc(o & (bit - 1));
        const int slot = (h >> 1) * 32 + (h & 1) * 16 + lane_in_half;
        os[slot] = s[i];
        od[slot] = d[i];
      }
    __syncthreads();
    // a dummy gathers what a neighbour gathers: every unused slot reading source
    // 0 would send one request per instruction to the same L2 sector from all
    // SMs (measured: 3 % dummies with source 0 halve K5's rate)
    if (tid < ni) {
      unsigned first = 0xffffffffu;
      for (int l = 0; l < 32 && first == 0xffffffffu; ++l)
        if (od[tid * 32 + l] != BR) first = os[tid * 32 + l];
      rownear[tid] = first;
    }
    __syncthreads();
    if (tid == 0) {
      unsigned near = 0u;
      for (int r = 0; r < ni; ++r)
        if (rownear[r] != 0xffffffffu) {
          near = rownear[r];
          break;
        }
      for (int r = 0; r < ni; ++r) {
        if (rownear[r] != 0xffffffffu) near = rownear[r];
        rownear[r] = near;
      }
    }
    __syncthreads();
    for (int i = tid; i < len; i += kBanksThreads) {
      const int p = blk_slot_pos(i);
      es[p] = od[i] != BR ? os[i] : rownear[i >> 5];
      ed[p] = od[i];
    }
    __syncthreads();
  }
}

// without the bank balance: slot order -> K5's lane-major order, chunk by chunk
__global__ void k_blk_lane_major(unsigned* __restrict__ esrc, unsigned short* __restrict__ edst, long long nchunks) {
  for (long long ch = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; ch < nchunks;
       ch += static_cast<long long>(gridDim.x) * blockDim.x) {
    unsigned* es = esrc + ch * kBlkChunk;
    unsigned short* ed = edst + ch * kBlkChunk;
    unsigned s[kBlkChunk];
    unsigned short d[kBlkChunk];
    for (int i = 0; i < kBlkChunk; ++i) {
      s[i] = es[i];
      d[i] = ed[i];
    }
    for (int i = 0; i < kBlkChunk; ++i) {
      es[blk_slot_pos(i)] = s[i];
      ed[blk_slot_pos(i)] = d[i];
    }
  }
}

int bits_for(long long v) {
  int b = 0;
  while ((1ll << b) < v) ++b;
  return b;
}

}  // namespace

cudaError_t build_blk_entries(const long long* iptr, const int* isrc, long long e_begin, long long E, int u0, int UR,
                              int row0, int R, int BR, const std::vector<long long>& pad_off, int slack, int win,
                              unsigned* esrc, unsigned short* edst, cudaStream_t s) {
  const int nb = static_cast<int>(pad_off.size()) - 1;
  const int sbits = std::max(1, bits_for(UR));
  const int end_bit = sbits + std::max(1, bits_for(nb));
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  long long* poff = nullptr;
  unsigned short *v0 = nullptr, *v1 = nullptr;
  void* tmp = nullptr;
  long long* wsd = nullptr;
  int* wld = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e = cudaSuccess;
  auto done = [&](cudaError_t r) {
    cudaStreamSynchronize(s);
    cudaFree(wsd);
    cudaFree(wld);
    cudaFree(k0);
    cudaFree(k1);
    cudaFree(v0);
    cudaFree(v1);
    cudaFree(tmp);
    cudaFree(poff);
    return r;
  };
  const size_t n = static_cast<size_t>(std::max<long long>(E, 1));
  if ((e = cudaMalloc(&k0, n * 8)) != cudaSuccess || (e = cudaMalloc(&k1, n * 8)) != cudaSuccess ||
      (e = cudaMalloc(&v0, n * 2)) != cudaSuccess || (e = cudaMalloc(&v1, n * 2)) != cudaSuccess ||
      (e = cudaMalloc(&poff, pad_off.size() * 8)) != cudaSuccess)
    return done(e);
  if ((e = cudaMemcpyAsync(poff, pad_off.data(), pad_off.size() * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return done(e);
  if (E > 0) {
    k_blk_keys<<<1184, 256, 0, s>>>(iptr, isrc, e_begin, u0, row0, R, BR, sbits, k0, v0);
    cub::DoubleBuffer<unsigned long long> kb(k0, k1);
    cub::DoubleBuffer<unsigned short> vb(v0, v1);
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, static_cast<std::int64_t>(E), 0, end_bit,
                                             s)) != cudaSuccess)
      return done(e);
    if ((e = cudaMalloc(&tmp, tmp_bytes)) != cudaSuccess) return done(e);
    if ((e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kb, vb, static_cast<std::int64_t>(E), 0, end_bit, s)) !=
        cudaSuccess)
      return done(e);
    k_blk_pack<<<2368, 256, 0, s>>>(iptr, e_begin, row0, R, BR, poff, nb, (1ull << sbits) - 1, kb.Current(),
                                    vb.Current(), esrc, edst, slack);
  } else {
    k_blk_pack<<<2368, 256, 0, s>>>(iptr, e_begin, row0, R, BR, poff, nb, (1ull << sbits) - 1, k0, v0, esrc, edst,
                                    slack);
  }
  if (win > 0) {  // windows never straddle blocks
    std::vector<long long> ws;
    std::vector<int> wl;
    for (int b = 0; b < nb; ++b)
      for (long long a = pad_off[static_cast<size_t>(b)]; a < pad_off[static_cast<size_t>(b) + 1]; a += win) {
        ws.push_back(a);
        wl.push_back(static_cast<int>(std::min<long long>(win, pad_off[static_cast<size_t>(b) + 1] - a)));
      }
    const long long nw = static_cast<long long>(ws.size());
    if ((e = cudaMalloc(&wsd, std::max<size_t>(1, ws.size()) * 8)) != cudaSuccess ||
        (e = cudaMalloc(&wld, std::max<size_t>(1, wl.size()) * 4)) != cudaSuccess ||
        (e = cudaMemcpyAsync(wsd, ws.data(), ws.size() * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(wld, wl.data(), wl.size() * 4, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return done(e);
    auto balance = [&](auto kern, int w) {
      const size_t smem = static_cast<size_t>(w) * 16 + static_cast<size_t>(w / 32) * 15;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      const char* er = std::getenv("LR_BLK_REACH");
      kern<<<static_cast<unsigned>(std::min<long long>(nw, 4 * 148)), kBanksThreads, smem, s>>>(esrc, edst, wsd, wld, nw, BR,
                                                                                   er ? std::atoi(er) : kBlkReach);
    };
    if (win == 256) balance(k_blk_banks<256>, 256);
    else if (win == 1024) balance(k_blk_banks<1024>, 1024);
    else if (win == 2048) balance(k_blk_banks<2048>, 2048);
    else if (win == 4096) balance(k_blk_banks<4096>, 4096);
    else balance(k_blk_banks<8192>, 8192);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return done(e);  // ws / wl are host temporaries
  } else if (!pad_off.empty() && pad_off.back() > 0) {
    k_blk_lane_major<<<1184, 128, 0, s>>>(esrc, edst, pad_off.back() / kBlkChunk);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return done(e);
  return done(cudaStreamSynchronize(s));
}

}  // namespace lrk
