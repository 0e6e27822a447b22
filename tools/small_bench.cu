// Microbenchmark of the SccSmall dense solve (K5) on synthetic SCCs:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --fmad=false \
//        -I include -I paper_1609_09068_b200/csrc/cuda tools/small_bench.cu -o build/small_bench
//   ./small_bench [m] [count]
// Times the production small_solve against the variants below, one CTA per
// SCC, and reports cycles per CTA (clock64) and the kernel time.
#define LR_TILE_PROBE
#include "../paper_1609_09068_b200/csrc/cuda/level.cu"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

namespace lrk {
namespace {

__global__ void __launch_bounds__(kThreads)
    k_bench_prod(DeviceLayout L, const SccTask* tasks, int ld, const double* pf, double* rank, DevStatus* st,
                 long long* cyc) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  const long long t0 = clock64();
  small_solve(L, tasks[blockIdx.x], ld, pf, rank, sm, red, st);
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

__global__ void __launch_bounds__(kThreads)
    k_bench_tile(DeviceLayout L, const SccTask* tasks, int ld, const double* pf, double* rank, DevStatus* st,
                 long long* cyc) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  const long long t0 = clock64();
  small_dispatch(L, tasks[blockIdx.x], ld, 0.85, pf, rank, sm, red, st);
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

}  // namespace
}  // namespace lrk

using namespace lrk;

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));      \
      std::exit(1);                                                               \
    }                                                                             \
  } while (0)

template <class T>
T* up(const std::vector<T>& v) {
  T* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!v.empty()) CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? std::atoi(argv[1]) : 64;
  const int K = argc > 2 ? std::atoi(argv[2]) : 256;
  const double c = 0.85;
  const int n = m * K;
  std::mt19937_64 rng(7);
  // each row: 6 in-edges from random other rows of its SCC (sorted sources)
  std::vector<long long> iptr(n + 1, 0);
  std::vector<int> isrc, deg(n, 0);
  for (int u = 0; u < K; ++u)
    for (int i = 0; i < m; ++i) {
      std::vector<int> srcs;
      for (int k = 0; k < 6 && m > 1; ++k) {
        int s = static_cast<int>(rng() % m);
        if (s == i) s = (s + 1) % m;
        srcs.push_back(u * m + s);
      }
      std::sort(srcs.begin(), srcs.end());
      srcs.erase(std::unique(srcs.begin(), srcs.end()), srcs.end());
      for (int s : srcs) {
        isrc.push_back(s);
        ++deg[s];
      }
      iptr[u * m + i + 1] = static_cast<long long>(isrc.size());
    }
  std::vector<double> pf(n), rank(n);
  for (int r = 0; r < n; ++r) {
    pf[r] = deg[r] ? c / (deg[r] + 2.0) : 0.0;  // +2: out-edges leaving the SCC
    rank[r] = 0.1 + (rng() % 1000) / 1000.0;
  }
  std::vector<SccTask> tasks(K);
  for (int u = 0; u < K; ++u) tasks[u] = SccTask{u * m, (u + 1) * m, u, 0, 0};
  std::vector<unsigned char> zeros(n, 0);
  DeviceLayout L{};
  L.n = n;
  L.iptr = up(iptr);
  L.isrc = up(isrc);
  L.deg = up(deg);
  L.loop = up(zeros);
  const double* d_pf = up(pf);
  double* d_rank0 = up(rank);
  double* d_rank;
  CK(cudaMalloc(&d_rank, n * sizeof(double)));
  const SccTask* d_tasks = up(tasks);
  DevStatus* st;
  CK(cudaMalloc(&st, sizeof(DevStatus)));
  CK(cudaMemset(st, 0, sizeof(DevStatus)));
  long long* cyc;
  CK(cudaMalloc(&cyc, K * sizeof(long long)));
  const int ld = m + 1;
  const size_t smem = static_cast<size_t>(ld) * (ld + 1) * sizeof(double);
  CK(cudaFuncSetAttribute(k_bench_prod, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(k_bench_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const size_t tsmem = m <= kSmallTileMaxM ? std::max(small_tile_bytes(m, static_cast<long long>(isrc.size() / K) + 64),
                                                      std::max(small_mma_bytes(static_cast<long long>(isrc.size() / K) + 64),
                                                               small_mma_smem_bytes(m, static_cast<long long>(isrc.size() / K) + 64)))
                                           : smem;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<double> out(n), ref(n);
  auto run = [&](const char* name, auto launch) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaMemcpy(d_rank, d_rank0, n * sizeof(double), cudaMemcpyDeviceToDevice));
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    std::vector<long long> h(K);
    CK(cudaMemcpy(h.data(), cyc, K * sizeof(long long), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out.data(), d_rank, n * sizeof(double), cudaMemcpyDeviceToHost));
    long long mx = 0, sum = 0;
    for (long long v : h) mx = std::max(mx, v), sum += v;
    double rel = 0.0;
    if (ref[0] == 0.0) ref = out;
    for (int i = 0; i < n; ++i) rel = std::max(rel, std::abs(out[i] - ref[i]) / std::abs(ref[i]));
    DevStatus hs;
    CK(cudaMemcpy(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost));
    CK(cudaMemset(st, 0, sizeof(DevStatus)));
    // host residual of (I - cA^T D^-1) x = w on the kernel's output
    double hres = 0.0;
    for (int r = 0; r < n; ++r) {
      double acc = out[r];
      for (long long e = iptr[r]; e < iptr[r + 1]; ++e) acc -= pf[isrc[e]] * out[isrc[e]];
      hres = std::max(hres, std::abs(acc - rank[r]) / std::abs(rank[r]));
    }
    std::printf("%-10s m=%d K=%d  %8.2f us  cycles/CTA avg %lld max %lld  rel=%.2e err=%u hostres=%.2e\n", name, m, K,
                best * 1e3, sum / K, mx, rel, hs.err, hres);
  };
  run("prod", [&] { k_bench_prod<<<K, kThreads, smem>>>(L, d_tasks, ld, d_pf, d_rank, st, cyc); });
  long long* probe;
  CK(cudaMalloc(&probe, static_cast<size_t>(K) * 160 * sizeof(long long)));
  CK(cudaMemcpyToSymbol(g_tile_probe, &probe, sizeof(probe)));
  run("tile", [&] { k_bench_tile<<<K, kThreads, tsmem>>>(L, d_tasks, ld, d_pf, d_rank, st, cyc); });
  std::vector<long long> hp(static_cast<size_t>(K) * 160);
  CK(cudaMemcpy(hp.data(), probe, hp.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  std::printf("  step cycles (CTA 0):");
  for (int k = 1; k < std::min(m, 24); ++k) std::printf(" %lld", hp[k] - hp[k - 1]);
  std::printf("\n");
  return 0;
}
