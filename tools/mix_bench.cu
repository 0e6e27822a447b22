// Do TMA tile::gather4 gathers add to the LDG gather rate, or share its limit
// (the SM's L1 -> XBAR request port)?  Each CTA runs LW warps of LDG gathers
// (ld.global.nc.L1::no_allocate, 8 per lane in flight) and TW warps of TMA
// gather4 (16-byte rows of the vector viewed as [n/2][2], lane 0 issuing 32
// gather4 per 128-row chunk, two chunks in flight).  The first f*m random
// indices go to the LDG warps, the rest to the TMA warps; the best f gives the
// combined rate.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/mix_bench.cu -o build/mix_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

__global__ void k_fill_idx(int* idx, long long m, unsigned n, unsigned long long seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = seed + 0x9E3779B97F4A7C15ull * (unsigned long long)(i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    idx[i] = (int)(z % n);
  }
}
__global__ void k_fill_x(double* x, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = 1.0 + (double)(i & 1023);
}
__device__ __forceinline__ int ld_idx(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_na(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void mbar_init(unsigned b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(unsigned b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned b, unsigned phase) {
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(b),
               "r"(phase)
               : "memory");
}
__device__ __forceinline__ void g4(unsigned dst, const CUtensorMap* tm, int r0, int r1, int r2, int r3, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(dst),
      "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}

__global__ void __launch_bounds__(1024) k_mix(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                              long long m_ldg, long long m, const double* __restrict__ x, int lw,
                                              double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc = 0.0;
  if (warp < lw) {
    constexpr int K = 8;
    const long long w = (long long)blockIdx.x * lw + warp, nw = (long long)gridDim.x * lw;
    for (long long c = w * 256; c + 256 <= m_ldg; c += nw * 256) {
      int id[K];
#pragma unroll
      for (int k = 0; k < K; ++k) id[k] = ld_idx(idx + c + lane + 32 * k);
      double g[K];
#pragma unroll
      for (int k = 0; k < K; ++k) g[k] = ld_na(x + id[k]);
#pragma unroll
      for (int k = 0; k < K; ++k) acc += g[k];
    }
  } else {
    const int tw = (blockDim.x >> 5) - lw, t = warp - lw;
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm);
    double2* stage = reinterpret_cast<double2*>(sm + 1024) + (size_t)t * 2 * 256;
    const unsigned b0 = (unsigned)__cvta_generic_to_shared(bars + 2 * t);
    const unsigned st0 = (unsigned)__cvta_generic_to_shared(stage);
    if (lane == 0) {
      mbar_init(b0, 1);
      mbar_init(b0 + 8, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const long long w = (long long)blockIdx.x * tw + t, W = (long long)gridDim.x * tw;
    int keep[2][4];
    auto issue = [&](long long c, int s) {
      int j[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) j[q] = idx[c + 4 * lane + q];
#pragma unroll
      for (int q = 0; q < 4; ++q) keep[s][q] = j[q];
      if (lane == 0) mbar_expect(b0 + 8 * s, 128 * 16);
      for (int l = 0; l < 32; ++l) {
        const int r0 = __shfl_sync(0xffffffffu, j[0], l) >> 1, r1 = __shfl_sync(0xffffffffu, j[1], l) >> 1;
        const int r2 = __shfl_sync(0xffffffffu, j[2], l) >> 1, r3 = __shfl_sync(0xffffffffu, j[3], l) >> 1;
        if (lane == 0) g4(st0 + (unsigned)(s * 32 + l) * 128u, &tm, r0, r1, r2, r3, b0 + 8 * s);
      }
    };
    unsigned ph = 0;
    long long c = m_ldg + w * 128;
    if (c + 128 <= m) issue(c, 0);
    int s = 0;
    while (c + 128 <= m) {
      const long long cn = c + W * 128;
      if (cn + 128 <= m) issue(cn, s ^ 1);
      mbar_wait(b0 + 8 * s, (ph >> s) & 1u);
      ph ^= 1u << s;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 v = stage[(s * 32 + lane) * 8 + q];
        acc += (keep[s][q] & 1) ? v.y : v.x;
      }
      __syncwarp();
      c = cn;
      s ^= 1;
    }
  }
  atomicAdd(out + 1, acc);
}

int main() {
  const long long m = 1ll << 27;
  const long long nmax = 21369371ll;
  int* idx;
  double *x, *out;
  CK(cudaMalloc(&idx, m * 4 + 4096));
  CK(cudaMalloc(&x, nmax * 8 + 64));
  CK(cudaMalloc(&out, 16));
  k_fill_x<<<1184, 256>>>(x, nmax);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const unsigned sizes[] = {4u << 20, 21369371u};
  CK(cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (unsigned n : sizes) {
    k_fill_idx<<<1184, 256>>>(idx, m, n, 12345);
    CK(cudaDeviceSynchronize());
    CUtensorMap tm;
    const cuuint64_t dims[2] = {2, (cuuint64_t)((n + 1) / 2)};
    const cuuint64_t strides[1] = {16};
    const cuuint32_t box[2] = {2, 1}, es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      std::printf("encode failed %d\n", (int)r);
      return 1;
    }
    std::printf("vector %u doubles (%.0f MB)\n", n, n * 8.0 / 1e6);
    const int cfg[][2] = {{24, 0}, {32, 0}, {0, 8}, {0, 16}, {24, 8}, {24, 4}, {16, 8}, {28, 4}};
    for (auto& cf : cfg) {
      const int lw = cf[0], tw = cf[1];
      const int threads = 32 * (lw + tw);
      const size_t smem = 1024 + (size_t)tw * 2 * 32 * 128;
      const double fs[] = {1.0, 0.9, 0.85, 0.8, 0.75, 0.7, 0.6, 0.0};
      for (double f : fs) {
        if ((tw == 0 && f < 1.0) || (lw == 0 && f > 0.0)) continue;
        long long ml = (long long)(f * m) & ~255ll;
        auto launch = [&] { k_mix<<<sms, threads, smem>>>(tm, idx, ml, m, x, lw, out); };
        launch();
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
          cudaEventRecord(e0);
          launch();
          cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        std::printf("  ldg warps %2d tma warps %2d f_ldg %.2f: %.3f ms  %.1f G gathers/s\n", lw, tw, f, best,
                    m / best / 1e6);
      }
    }
  }
  return 0;
}
