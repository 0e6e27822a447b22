// Latency probes (cycles) on the running GPU: dependent FP64 multiply/add,
// dependent shared-memory load, CTA barrier, IEEE double reciprocal.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false tools/lat_bench.cu -o build/lat_bench
#include <cstdio>

__global__ void k_probe(double* out, long long* cyc, double seed) {
  __shared__ int chase[256];
  __shared__ double dsm[256];
  const int tid = threadIdx.x;
  chase[tid] = (tid + 1) & 255;
  dsm[tid] = seed + tid;
  __syncthreads();
  double x = seed + tid;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = x * 1.0000001;
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = x + 1e-9;
  long long t2 = clock64();
  int p = tid;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) p = chase[p];
  long long t3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) __syncthreads();
  long long t4 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) x = 1.0 / x;
  long long t5 = clock64();
  double y = dsm[tid];
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {  // LDS -> DMUL -> STS -> barrier: one GJ-like step
    __syncthreads();
    y = dsm[(tid + i) & 255] * 1.0000001;
    dsm[tid] = y;
  }
  long long t6 = clock64();
  out[tid] = x + p + y;
  if (tid == 0) {
    cyc[0] = (t1 - t0) / 256;
    cyc[1] = (t2 - t1) / 256;
    cyc[2] = (t3 - t2) / 256;
    cyc[3] = (t4 - t3) / 256;
    cyc[4] = (t5 - t4) / 64;
    cyc[5] = (t6 - t5) / 256;
  }
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 256 * sizeof(double));
  cudaMalloc(&cyc, 8 * sizeof(long long));
  for (int rep = 0; rep < 2; ++rep) k_probe<<<1, 256>>>(out, cyc, 1.5);
  long long h[8];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  std::printf("DMUL %lld  DADD %lld  LDS-chase %lld  bar.sync(256) %lld  1.0/x %lld  bar+LDS+DMUL+STS %lld cycles\n",
              h[0], h[1], h[2], h[3], h[4], h[5]);
  return 0;
}
