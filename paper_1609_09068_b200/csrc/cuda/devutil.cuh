// Small device helpers shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdio>

// Device-side bounds checks of the gathers (compute-sanitizer is closed on the
// GPU pool): build with -DLR_DEVICE_CHECKS (tools/build_variant.sh dchecks
// -DLR_DEVICE_CHECKS) and run the GPU suite with LR_LIB pointing at it; a failed
// check prints its site and traps the kernel.  Compiled out otherwise.
#ifdef LR_DEVICE_CHECKS
#define LR_DCHECK(cond)                                                                     \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("LR_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                 \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define LR_DCHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace lrk {
namespace dev {

__device__ __forceinline__ unsigned long long dbits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}
__device__ __forceinline__ double bitsd(unsigned long long b) {
  return __longlong_as_double(static_cast<long long>(b));
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// Fixed butterfly order: deterministic for a given lane assignment.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Block-wide max / sum; `red` holds blockDim/32 doubles; all threads get the result.
__device__ __forceinline__ double block_max(double v, double* red) {
  v = warp_max(v);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) red[warp] = v;
  __syncthreads();
  double m = red[0];
  for (int i = 1; i < nw; ++i) m = fmax(m, red[i]);
  return m;
}
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) red[warp] = v;
  __syncthreads();
  double s = red[0];
  for (int i = 1; i < nw; ++i) s += red[i];
  return s;
}

}  // namespace dev
}  // namespace lrk
