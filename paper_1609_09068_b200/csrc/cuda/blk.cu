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
// the work is split by slots, not by blocks)
__global__ void k_blk_pack(const long long* __restrict__ iptr, long long e_begin, int u0, int R, int BR,
                           const long long* __restrict__ pad_off, int nb, unsigned long long smask,
                           const unsigned long long* __restrict__ keys, const unsigned short* __restrict__ vals,
                           unsigned* __restrict__ esrc, unsigned short* __restrict__ edst) {
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
    const long long j = i - pad_off[lo];
    if (j < cnt) {
      esrc[i] = static_cast<unsigned>(keys[s0 + j] & smask);
      edst[i] = vals[s0 + j];
    } else {
      esrc[i] = 0u;
      edst[i] = static_cast<unsigned short>(BR);
    }
  }
}

// Shared-memory bank balance of each 256-entry chunk (one thread per chunk).
// K5 lane l of a warp handles entries l + 32 k; its atomic add to y[dst] hits
// the bank pair dst mod 16 (8-byte words), and a half-warp whose 16 adds use
// 16 distinct bank pairs takes one shared-memory wavefront (random dsts: ~5 per
// instruction; measured 2 vs 4 adds per SM-clock, tools/atoms_bench.cu).  Walk
// the chunk in source order and put each entry into the half-warp nearest its
// own whose slot for that bank pair is free (else the nearest half with room),
// so each gather instruction still reads sources from about the same lines.
__global__ void k_blk_banks(unsigned* __restrict__ esrc, unsigned short* __restrict__ edst, long long nchunks) {
  for (long long ch = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; ch < nchunks;
       ch += static_cast<long long>(gridDim.x) * blockDim.x) {
    unsigned* es = esrc + ch * kBlkChunk;
    unsigned short* ed = edst + ch * kBlkChunk;
    unsigned s[kBlkChunk];
    unsigned short d[kBlkChunk];
    unsigned char to[kBlkChunk];
    for (int i = 0; i < kBlkChunk; ++i) {
      s[i] = es[i];
      d[i] = ed[i];
    }
    unsigned short occ[16] = {};
    unsigned char fill[16] = {};
    for (int i = 0; i < kBlkChunk; ++i) {
      const int c = d[i] & 15, h0 = i >> 4;
      int best = -1;
      for (int dist = 0; dist < 16 && best < 0; ++dist)
        for (int sg = 0; sg < 2 && best < 0; ++sg) {
          const int h = sg ? h0 - dist : h0 + dist;
          if ((sg && dist == 0) || h < 0 || h > 15) continue;
          if (fill[h] < 16 && !((occ[h] >> c) & 1)) best = h;
        }
      for (int dist = 0; dist < 16 && best < 0; ++dist)
        for (int sg = 0; sg < 2 && best < 0; ++sg) {
          const int h = sg ? h0 - dist : h0 + dist;
          if ((sg && dist == 0) || h < 0 || h > 15) continue;
          if (fill[h] < 16) best = h;
        }
      occ[best] = static_cast<unsigned short>(occ[best] | (1u << c));
      to[i] = static_cast<unsigned char>((best >> 1) * 32 + (best & 1) * 16 + fill[best]++);
    }
    for (int i = 0; i < kBlkChunk; ++i) {
      es[to[i]] = s[i];
      ed[to[i]] = d[i];
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
                              int BR, const std::vector<long long>& pad_off, unsigned* esrc, unsigned short* edst,
                              cudaStream_t s) {
  const int nb = static_cast<int>(pad_off.size()) - 1;
  const int sbits = std::max(1, bits_for(R));
  const int end_bit = sbits + std::max(1, bits_for(nb));
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  long long* poff = nullptr;
  unsigned short *v0 = nullptr, *v1 = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e = cudaSuccess;
  auto done = [&](cudaError_t r) {
    cudaStreamSynchronize(s);
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
    k_blk_pack<<<2368, 256, 0, s>>>(iptr, e_begin, u0, R, BR, poff, nb, (1ull << sbits) - 1,
                                                  kb.Current(), vb.Current(), esrc, edst);
  } else {
    k_blk_pack<<<2368, 256, 0, s>>>(iptr, e_begin, u0, R, BR, poff, nb, (1ull << sbits) - 1, k0, v0,
                                                  esrc, edst);
  }
  {
    const char* eb = std::getenv("LR_BLK_BANKS");
    if (!(eb && std::atoi(eb) == 0))
      k_blk_banks<<<1184, 128, 0, s>>>(esrc, edst, pad_off.back() / kBlkChunk);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return done(e);
  return done(cudaStreamSynchronize(s));
}

}  // namespace lrk
