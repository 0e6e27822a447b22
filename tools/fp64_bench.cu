// FP64 FMA throughput and latency on the running GPU (the small-SCC eliminations
// and CTA power series are chains of dependent FP64 operations):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_bench.cu -o build/fp64_bench
#include <cstdio>

template <int CHAINS>
__global__ void k_fma(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __fma_rn(x[c], a, b);
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 1 << 14;
  auto run = [&](auto kern, int chains, int blocks, int threads) {
    kern<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = double(blocks) * threads * iters * chains;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    std::printf("chains %d blocks %d threads %d: %.3f ms  %.2f TFMA/s  %.1f FMA/clk/SM (at %d MHz nominal)\n", chains,
                blocks, threads, ms, fmas / ms / 1e9, fmas / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000);
  };
  run(k_fma<1>, 1, 1, 32);        // latency: one warp, one chain
  run(k_fma<8>, 8, 1, 32);        // one warp, 8 chains
  run(k_fma<8>, 8, sms, 256);     // 8 warps per SM
  run(k_fma<8>, 8, sms * 4, 256); // 32 warps per SM
  run(k_fma<4>, 4, sms * 8, 256);
  return 0;
}
