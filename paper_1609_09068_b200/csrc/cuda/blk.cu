// Device-side build of K5's dest-blocked layout (kernels.cuh BlkUnitDev) from
// the unit's in-edge CSR already on the device: key every in-edge by
// (dest block, source), radix-sort the keys with the in-block dest row as
// payload (CUB, one-time setup at upload), then scatter each block's sorted run
// into its padded slot, dummies (src 0, dst BR) in the padding.  Rows are in
// unit order, so block b's in-edges occupy the same CSR range before and after
// the sort: the sort only reorders inside blocks.
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
                           int R, int BR, int sbits, unsigned long long* __restrict__ keys,
                           unsigned short* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const long long w0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long r = w0; r < R; r += nw) {
    const long long g = u0 + r;
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
__global__ void k_blk_pack(const long long* __restrict__ iptr, long long e_begin, int u0, int R, int BR,
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
    const long long s0 = iptr[u0 + r0] - e_begin, cnt = iptr[u0 + r1] - iptr[u0 + r0];
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

// Shared-memory bank balance, one thread per window of W slots (several chunks
// of one block).  K5 lane l of a warp handles slots l + 32 k of a chunk; its
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
template <int W>
__global__ void k_blk_banks(unsigned* __restrict__ esrc, unsigned short* __restrict__ edst,
                            const long long* __restrict__ wstart, const int* __restrict__ wlen, long long nwin,
                            int BR) {
  constexpr int G = W / 16;
  for (long long wi = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; wi < nwin;
       wi += static_cast<long long>(gridDim.x) * blockDim.x) {
    unsigned* es = esrc + wstart[wi];
    unsigned short* ed = edst + wstart[wi];
    const int len = wlen[wi], ni = len / 32;
    unsigned s[W];
    unsigned short d[W], to[W], left[W];
    unsigned short occ[G];
    unsigned char fill[G];
    for (int i = 0; i < len; ++i) {
      s[i] = es[i];
      d[i] = ed[i];
      es[i] = 0u;
      ed[i] = static_cast<unsigned short>(BR);
    }
    for (int h = 0; h < 2 * ni; ++h) occ[h] = 0, fill[h] = 0;
    auto put = [&](int i, int h) {
      occ[h] = static_cast<unsigned short>(occ[h] | (1u << (d[i] & 15)));
      to[i] = static_cast<unsigned short>((h >> 1) * 32 + (h & 1) * 16 + fill[h]++);
    };
    int nleft = 0;
    for (int i = 0; i < len; ++i) {
      if (d[i] == BR) continue;  // a dummy: its slot is free
      const int c = d[i] & 15, a = (i >> 5) * 2;
      if (!((occ[a] >> c) & 1)) put(i, a);
      else if (!((occ[a + 1] >> c) & 1)) put(i, a + 1);
      else left[nleft++] = static_cast<unsigned short>(i);
    }
    int nrest = 0;
    for (int q = 0; q < nleft; ++q) {
      const int i = left[q], c = d[i] & 15, i0 = i >> 5;
      int best = -1;
      for (int dist = 1; dist < ni && best < 0; ++dist)
        for (int sg = 0; sg < 2 && best < 0; ++sg) {
          const int in = sg ? i0 - dist : i0 + dist;
          if (in < 0 || in >= ni) continue;
          for (int h = 2 * in; h < 2 * in + 2 && best < 0; ++h)
            if (fill[h] < 16 && !((occ[h] >> c) & 1)) best = h;
        }
      if (best < 0) left[nrest++] = static_cast<unsigned short>(i);
      else put(i, best);
    }
    for (int q = 0; q < nrest; ++q) {
      const int i = left[q], i0 = i >> 5;
      int best = -1;
      for (int dist = 0; dist < ni && best < 0; ++dist)
        for (int sg = 0; sg < 2 && best < 0; ++sg) {
          const int in = sg ? i0 - dist : i0 + dist;
          if ((sg && dist == 0) || in < 0 || in >= ni) continue;
          for (int h = 2 * in; h < 2 * in + 2 && best < 0; ++h)
            if (fill[h] < 16) best = h;
        }
      put(i, best);
    }
    for (int i = 0; i < len; ++i)
      if (d[i] != BR) {
        es[to[i]] = s[i];
        ed[to[i]] = d[i];
      }
    // a dummy gathers what a neighbour gathers: every unused slot reading source
    // 0 would send one request per instruction to the same L2 sector from all
    // SMs (measured: 3 % dummies with source 0 halve K5's rate)
    unsigned near = 0u;
    for (int i = 0; i < len && near == 0u; ++i)
      if (d[i] != BR) near = s[i];
    for (int r = 0; r < ni; ++r) {
      for (int l = 0; l < 32; ++l)
        if (ed[r * 32 + l] != BR) {
          near = es[r * 32 + l];
          break;
        }
      for (int l = 0; l < 32; ++l)
        if (ed[r * 32 + l] == BR) es[r * 32 + l] = near;
    }
  }
}

int bits_for(long long v) {
  int b = 0;
  while ((1ll << b) < v) ++b;
  return b;
}

}  // namespace

cudaError_t build_blk_entries(const long long* iptr, const int* isrc, long long e_begin, long long E, int u0, int R,
                              int BR, const std::vector<long long>& pad_off, int slack, int win, unsigned* esrc,
                              unsigned short* edst, cudaStream_t s) {
  const int nb = static_cast<int>(pad_off.size()) - 1;
  const int sbits = std::max(1, bits_for(R));
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
    k_blk_keys<<<1184, 256, 0, s>>>(iptr, isrc, e_begin, u0, R, BR, sbits, k0, v0);
    cub::DoubleBuffer<unsigned long long> kb(k0, k1);
    cub::DoubleBuffer<unsigned short> vb(v0, v1);
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, static_cast<std::int64_t>(E), 0, end_bit,
                                             s)) != cudaSuccess)
      return done(e);
    if ((e = cudaMalloc(&tmp, tmp_bytes)) != cudaSuccess) return done(e);
    if ((e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kb, vb, static_cast<std::int64_t>(E), 0, end_bit, s)) !=
        cudaSuccess)
      return done(e);
    k_blk_pack<<<2368, 256, 0, s>>>(iptr, e_begin, u0, R, BR, poff, nb, (1ull << sbits) - 1, kb.Current(),
                                    vb.Current(), esrc, edst, slack);
  } else {
    k_blk_pack<<<2368, 256, 0, s>>>(iptr, e_begin, u0, R, BR, poff, nb, (1ull << sbits) - 1, k0, v0, esrc, edst,
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
    if (win == 256) k_blk_banks<256><<<592, 64, 0, s>>>(esrc, edst, wsd, wld, nw, BR);
    else if (win == 1024) k_blk_banks<1024><<<592, 64, 0, s>>>(esrc, edst, wsd, wld, nw, BR);
    else if (win == 2048) k_blk_banks<2048><<<592, 64, 0, s>>>(esrc, edst, wsd, wld, nw, BR);
    else if (win == 4096) k_blk_banks<4096><<<592, 32, 0, s>>>(esrc, edst, wsd, wld, nw, BR);
    else k_blk_banks<8192><<<592, 32, 0, s>>>(esrc, edst, wsd, wld, nw, BR);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return done(e);  // ws / wl are host temporaries
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return done(e);
  return done(cudaStreamSynchronize(s));
}

}  // namespace lrk
