// Shared-memory fp64 accumulation rates on the running GPU: random
// y[d] += v into a per-CTA array of BR doubles (atomicAdd on shared doubles
// compiles to an LDS + DADD + ATOMS.CAST.SPIN.64 loop on sm_100a), against
// plain random STS and LDS, 148 CTAs x T threads, 8 independent updates per
// thread in flight.  Decides whether a dest-blocked SpMV can accumulate its
// rows with shared-memory atomics.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/atoms_bench.cu -o build/atoms_bench
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

template <int MODE>
__global__ void k(int iters, int br, double* out) {
  extern __shared__ double y[];
  for (int i = threadIdx.x; i < br; i += blockDim.x) y[i] = 0.0;
  __syncthreads();
  unsigned s = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    unsigned d[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      s = s * 1664525u + 1013904223u;
      d[q] = (s >> 8) % br;
      if (MODE == 3 || MODE == 4) d[q] = (d[q] & ~15u) | (threadIdx.x & 15u);  // each half-warp: 16 distinct bank pairs
      if (MODE >= 5) d[q] = (d[q] & ~31u) | (threadIdx.x & 31u);  // and 32 distinct rows per warp instruction
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (MODE == 0 || MODE == 3) atomicAdd(&y[d[q]], 1.0 + q);
      if (MODE == 4) acc += y[d[q]];
      if (MODE == 1) y[d[q]] = 1.0 + q;
      if (MODE == 2) acc += y[d[q]];
      if (MODE == 5) {  // take the row (exchange with a sentinel), add, put it back
        unsigned long long* a = reinterpret_cast<unsigned long long*>(&y[d[q]]);
        unsigned long long old;
        do old = atomicExch(a, ~0ull);
        while (old == ~0ull);
        *reinterpret_cast<volatile double*>(a) = __longlong_as_double(static_cast<long long>(old)) + (1.0 + q);
      }
      if (MODE == 6) {  // not atomic: the lower bound (LDS + DADD + STS)
        volatile double* a = &y[d[q]];
        *a = *a + (1.0 + q);
      }
    }
  }
  __syncthreads();
  double t = acc;
  for (int i = threadIdx.x; i < br; i += blockDim.x) t += y[i];
  if (t == -1.0) out[0] = t;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[7] = {"atomicAdd f64 (CAS loop)", "random STS.64", "random LDS.64", "atomicAdd, no conflicts",
                          "LDS.64, no conflicts", "exchange-lock add, no conflicts", "LDS+DADD+STS, no conflicts"};
  for (int mode = 0; mode < 7; ++mode)
    for (int threads : {1024})
      for (int br : {16384}) {
        const size_t smem = br * 8;
        const int iters = 2000;
        auto launch = [&] {
          if (mode == 0) k<0><<<sms, threads, smem>>>(iters, br, out);
          if (mode == 1) k<1><<<sms, threads, smem>>>(iters, br, out);
          if (mode == 2) k<2><<<sms, threads, smem>>>(iters, br, out);
          if (mode == 3) k<3><<<sms, threads, smem>>>(iters, br, out);
          if (mode == 4) k<4><<<sms, threads, smem>>>(iters, br, out);
          if (mode == 5) k<5><<<sms, threads, smem>>>(iters, br, out);
          if (mode == 6) k<6><<<sms, threads, smem>>>(iters, br, out);
        };
        CK(cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CK(cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CK(cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CK(cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CK(cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CK(cudaFuncSetAttribute(k<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CK(cudaFuncSetAttribute(k<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        launch();
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
          cudaEventRecord(e0);
          launch();
          cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        const double ops = (double)sms * threads * iters * 8;
        std::printf("%-26s %4d thr  y %5d: %.3f ms  %.1f G ops/s  %.2f ops/SM-clk@1.9GHz\n", names[mode], threads, br,
                    best, ops / best / 1e6, ops / best / 1e6 / sms / 1.9);
      }
  return 0;
}
