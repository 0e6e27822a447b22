// lr_ctx: device residency of one Layout and the stream-ordered level loop
// (the GPU replacement of compute_pagerank's loop, proj/src/engine.cpp:126-158).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "kernels.cuh"
#include "lr_cuda.h"

#include <dlfcn.h>
#include <nccl.h>  // types only; the library is resolved at run time (see nccl())

namespace lrerr {
void set(const std::string& msg);
}

using namespace lrk;

namespace {

#define LR_CUDA_TRY(expr)                                                                          \
  do {                                                                                             \
    const cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) {                                                                       \
      lrerr::set(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #expr);             \
      return e_ == cudaErrorMemoryAllocation ? LR_ENOMEM : LR_ECUDA;                               \
    }                                                                                              \
  } while (0)

// Copies between large pageable host arrays and the device (the layout's index
// arrays, a caller's std::vector of weights or ranks): the runtime stages such a
// copy through its own pinned buffer with one thread (~10 GB/s); here four
// threads move 32 MB pinned buffers in turn while the neighbouring ones are on
// the wire (PCIe 5: ~55 GB/s).  Small copies, pinned callers and failures to get
// pinned memory take the plain path.
namespace {
constexpr size_t kStageChunk = size_t{32} << 20;
constexpr int kStageBufs = 4, kStageThreads = 4;
struct Stage {
  void* buf[kStageBufs] = {};
  cudaEvent_t ev[kStageBufs] = {};
  bool ok = false;
  Stage() {
    for (int i = 0; i < kStageBufs; ++i)
      if (cudaHostAlloc(&buf[i], kStageChunk, cudaHostAllocPortable) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return;
      }
    ok = true;
  }
};
std::mutex g_stage_mu;  // one staged copy at a time (the buffers are shared by every context of a device)
// the current device's staging buffers (events belong to the device that created them); call under g_stage_mu
Stage* stage_for_device() {
  constexpr int kMaxDev = 64;
  static std::unique_ptr<Stage> stages[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  if (!stages[dev]) stages[dev] = std::make_unique<Stage>();
  return stages[dev]->ok ? stages[dev].get() : nullptr;
}
void parallel_memcpy(void* dst, const void* src, size_t len) {
  std::thread th[kStageThreads - 1];
  const size_t piece = (len + kStageThreads - 1) / kStageThreads;
  for (int t = 1; t < kStageThreads; ++t)
    th[t - 1] = std::thread([=] {
      const size_t lo = std::min(len, piece * t), hi = std::min(len, piece * (t + 1));
      std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
    });
  std::memcpy(dst, src, std::min(len, piece));
  for (auto& t : th) t.join();
}
bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}
}  // namespace

static cudaError_t h2d_async(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes < 2 * kStageChunk || host_pinned(src)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  std::lock_guard<std::mutex> lock(g_stage_mu);
  Stage* st = stage_for_device();
  if (!st) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  const char* from = static_cast<const char*>(src);
  char* to = static_cast<char*>(dst);
  cudaError_t e = cudaSuccess;
  size_t i = 0;
  for (size_t off = 0; off < bytes && e == cudaSuccess; off += kStageChunk, ++i) {
    const int b = static_cast<int>(i % kStageBufs);
    const size_t len = std::min(kStageChunk, bytes - off);
    if (i >= kStageBufs && (e = cudaEventSynchronize(st->ev[b])) != cudaSuccess) break;
    parallel_memcpy(st->buf[b], from + off, len);
    if ((e = cudaMemcpyAsync(to + off, st->buf[b], len, cudaMemcpyHostToDevice, s)) != cudaSuccess) break;
    e = cudaEventRecord(st->ev[b], s);
  }
  // the buffers may be reused by another stream next: drain them before unlocking
  for (int b = 0; b < kStageBufs && b < static_cast<int>(i); ++b) {
    const cudaError_t w = cudaEventSynchronize(st->ev[b]);
    if (e == cudaSuccess && w != cudaSuccess) e = w;
  }
  return e;
}

// device -> pageable host, complete on return
static cudaError_t d2h_sync(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  auto plain = [&] {
    const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
    return e != cudaSuccess ? e : cudaStreamSynchronize(s);
  };
  if (bytes < 2 * kStageChunk || host_pinned(dst)) return plain();
  std::lock_guard<std::mutex> lock(g_stage_mu);
  Stage* st = stage_for_device();
  if (!st) return plain();
  const char* from = static_cast<const char*>(src);
  char* to = static_cast<char*>(dst);
  const size_t nchunks = (bytes + kStageChunk - 1) / kStageChunk;
  cudaError_t e = cudaSuccess;
  auto drain = [&](size_t j) {  // chunk j: wait for its copy, then move it out of the pinned buffer
    const int b = static_cast<int>(j % kStageBufs);
    if ((e = cudaEventSynchronize(st->ev[b])) != cudaSuccess) return;
    const size_t off = j * kStageChunk;
    parallel_memcpy(to + off, st->buf[b], std::min(kStageChunk, bytes - off));
  };
  for (size_t i = 0; i < nchunks && e == cudaSuccess; ++i) {
    if (i >= kStageBufs) drain(i - kStageBufs);  // frees buffer i % kStageBufs
    if (e != cudaSuccess) break;
    const int b = static_cast<int>(i % kStageBufs);
    const size_t off = i * kStageChunk;
    if ((e = cudaMemcpyAsync(st->buf[b], from + off, std::min(kStageChunk, bytes - off), cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
    e = cudaEventRecord(st->ev[b], s);
  }
  for (size_t j = nchunks > kStageBufs ? nchunks - kStageBufs : 0; j < nchunks && e == cudaSuccess; ++j) drain(j);
  if (e != cudaSuccess) cudaStreamSynchronize(s);
  return e;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  cudaError_t alloc(size_t count) {
    reset();
    n = count;
    return cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
  }
  cudaError_t upload(const T* src, size_t count, cudaStream_t s) {
    cudaError_t e = alloc(count);
    if (e != cudaSuccess || count == 0) return e;
    return h2d_async(p, src, count * sizeof(T), s);
  }
  cudaError_t upload_padded(const T* src, size_t count, size_t pad, cudaStream_t s) {
    cudaError_t e = alloc(count + pad);
    n = count;
    if (e != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(p + count, 0, pad * sizeof(T), s)) != cudaSuccess || count == 0) return e;
    return h2d_async(p, src, count * sizeof(T), s);
  }
  size_t bytes() const { return n * sizeof(T); }
};

struct LevelTasks {
  int rb = 0, re = 0;
  int cac_w0 = 0, cac_w1 = 0;  // warp-per-CAC tasks
  int cac_m0 = 0, cac_m1 = 0;  // 256-thread CTA per CAC (k_level)
  int cac_b0 = 0, cac_b1 = 0;  // 1024-thread CTA per CAC (side stream)
  int sm0 = 0, sm1 = 0, sm_max = 0;
  int lc0 = 0, lc1 = 0, lc_max = 0;
  int xh0 = 0, xh1 = 0;  // split cross rows (more than kCrossSplit in-edges)
  int sb0 = 0, sb1 = 0, sb_max = 0;  // SccSmall units beyond shared memory
  int lt0 = 0, lt1 = 0;  // CTA tasks of the fused level kernel
  int xb0 = 0, xb1 = 0;  // row tasks: start weights of the level's largest k_cac_big CACs (side stream)
  bool xb_fin = false;   // ... split: kTaskRowsFin tasks finishing sums begun one level earlier
  int pt0 = 0, pt1 = 0;  // kTaskRowsPart tasks for the NEXT level's large CACs (pre stream, this level)
  size_t smem = 0;       // its dynamic shared memory
  size_t big_smem = 0;   // dynamic shared memory of the k_cac_big launch
  size_t sm_tile = 0;    // largest small_solve_tile footprint of the level
  int sl0 = 0, sl1 = 0;  // depth slices of large CACs (one launch each)
  int gu0 = 0, gu1 = 0;
  int bk0 = 0, bk1 = 0;
  // L2 residency of the largest grid unit's pushed vectors: rows
  // [hot_begin, hot_begin + hot_rows) evict-last, the rest of the unit evict-first
  int hot_begin = 0;
  long long hot_rows = 0, unit_rows = 0;
  int keep_stream = 0;  // L2 priority of the streamed SpMV operands (spmv.cu policy_stream)
  int blk = -1;         // K5: index into lr_ctx::blk (the level's one grid unit by dest-row blocks), or -1
  std::vector<int> blk_chunks;  // row-sharded: the same per exchange chunk of this rank's shard (-1: K4c)
  // multi-GPU, large levels: rows split over the ranks for the CTA-solved
  // units (world + 1 bounds; empty = every rank solves the whole level)
  std::vector<int> dist_bounds;
  // multi-GPU, one grid unit on the level: this rank's blocks per exchange
  // chunk ([chunk_bk[j], chunk_bk[j+1]) relative to the level's blocks)
  std::vector<int> chunk_bk;
};

// One depth slice of a large CAC: rows [r0, r1), heavy-row tasks [h0, h1).
struct CacSlice {
  int r0, r1, h0, h1;
};

// NCCL, resolved with dlopen so the library loads (and every single-GPU path
// works) where NCCL is absent; in a torch process this binds to the libnccl.so.2
// torch already loaded.
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.broadcast = reinterpret_cast<decltype(a.broadcast)>(dlsym(h, "ncclBroadcast"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.broadcast && a.all_reduce && a.group_start &&
           a.group_end && a.error_string;
    return a;
  }();
  return api;
}

#define LR_NCCL_TRY(expr)                                                                          \
  do {                                                                                             \
    const ncclResult_t r_ = (expr);                                                                \
    if (r_ != ncclSuccess) {                                                                       \
      lrerr::set(std::string("NCCL error: ") + nccl().error_string(r_) + " at " #expr);            \
      return LR_ENCCL;                                                                             \
    }                                                                                              \
  } while (0)

// nnz-balanced contiguous split of rows [rb, re) over `world` parts (iptr is
// the row-pointer array of the whole layout).
std::vector<int> shard_bounds(const int64_t* iptr, int rb, int re, int world) {
  std::vector<int> b(static_cast<size_t>(world) + 1, rb);
  const long long e0 = iptr[rb], total = iptr[re] - e0;
  for (int r = 1; r < world; ++r) {
    const long long target = e0 + total * r / world;
    b[static_cast<size_t>(r)] = static_cast<int>(std::lower_bound(iptr + rb, iptr + re, target) - iptr);
  }
  b[static_cast<size_t>(world)] = re;
  for (int r = 1; r <= world; ++r) b[static_cast<size_t>(r)] = std::max(b[static_cast<size_t>(r)], b[static_cast<size_t>(r) - 1]);
  return b;
}

// Exchange chunks of a row-sharded unit: rank q's shard [b_q, b_{q+1}) cut
// into `chunks` nnz-balanced pieces of whole rows; world * chunks + 1 bounds,
// rank q's chunk j = [cuts[q * chunks + j], cuts[q * chunks + j + 1]).  Every
// rank computes the same cuts from the same layout.
std::vector<int> exchange_cuts(const int64_t* iptr, int rb, int re, int world, int chunks) {
  const std::vector<int> b = shard_bounds(iptr, rb, re, world);
  std::vector<int> cuts;
  cuts.reserve(static_cast<size_t>(world) * static_cast<size_t>(chunks) + 1);
  for (int q = 0; q < world; ++q) {
    const std::vector<int> c = shard_bounds(iptr, b[static_cast<size_t>(q)], b[static_cast<size_t>(q) + 1], chunks);
    cuts.insert(cuts.end(), c.begin(), c.end() - 1);
  }
  cuts.push_back(re);
  return cuts;
}

// Rows of one level split over `world` ranks for the level's CTA-solved units
// (multi-GPU, lr_split_level_rows): contiguous row ranges balanced by a cost
// of rows + cross in-edges + intra in-edges (x32 for units small enough for
// the CTA power series, whose edges are walked every iteration); singleton
// groups and grid units are cut anywhere (their rows are independent row
// tasks), every other unit is kept whole.  world + 1 bounds.
std::vector<int> split_level_rows(const int64_t* iptr, const int64_t* xptr, const int32_t* unit_row_begin,
                                  const std::uint8_t* unit_kind, int u0, int u1, int world) {
  const int rb = unit_row_begin[u0], re = unit_row_begin[u1];
  std::vector<int> b(static_cast<size_t>(world) + 1, rb);
  b[static_cast<size_t>(world)] = re;
  if (world <= 1 || re <= rb) return b;
  auto cost = [&](int u) {
    const int a = unit_row_begin[u], e = unit_row_begin[u + 1];
    const long long intra = iptr[e] - iptr[a];
    const bool cta_series = unit_kind[u] == 3 && e - a <= kCtaLargeMaxRows && intra <= kCtaLargeMaxNnz;
    return static_cast<double>(e - a) + static_cast<double>(xptr[e] - xptr[a]) +
           static_cast<double>(intra) * (cta_series ? 32.0 : 1.0);
  };
  double total = 0.0;
  for (int u = u0; u < u1; ++u) total += cost(u);
  double acc = 0.0;
  int q = 1;
  for (int u = u0; u < u1 && q < world; ++u) {
    const int a = unit_row_begin[u], e = unit_row_begin[u + 1];
    const double c = cost(u);
    const bool divisible = unit_kind[u] == 0 ||
                           (unit_kind[u] == 3 && !(e - a <= kCtaLargeMaxRows && iptr[e] - iptr[a] <= kCtaLargeMaxNnz));
    while (q < world && acc + c >= total * q / world) {
      const double target = total * q / world;
      int cut = e;
      if (divisible && e > a) {
        const double per_row = c / static_cast<double>(e - a);
        cut = a + static_cast<int>(std::ceil((target - acc) / per_row));
        cut = std::min(std::max(cut, a), e);
      } else if (target - acc < acc + c - target) {
        cut = a;
      }
      b[static_cast<size_t>(q)] = std::max(cut, b[static_cast<size_t>(q) - 1]);
      ++q;
    }
    acc += c;
  }
  for (; q < world; ++q) b[static_cast<size_t>(q)] = re;
  return b;
}

}  // namespace

struct lr_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // runs of levels without grid SpMV units, captured once into CUDA graphs and
  // replayed every solve (their launches depend on nothing the host decides)
  struct Segment {
    int begin, end;          // levels [begin, end)
    int64_t launches;        // kernel launches inside
    cudaGraphExec_t exec;
  };
  std::vector<Segment> segs;
  bool segs_built = false;
  void drop_graphs() {
    for (auto& g : segs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    segs.clear();
    segs_built = false;
  }
  cudaStream_t side = nullptr;  // large CACs, concurrent with each level's k_level
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  // early partial start-weight sums of the next level's large CACs (kTaskRowsPart)
  cudaStream_t pre = nullptr;
  cudaEvent_t pre_fork = nullptr, pre_done = nullptr;
  DevBuf<double> xpart;
  int n = 0;
  int n_levels = 0;
  int64_t n_units = 0;
  bool loaded = false;
  std::vector<LevelTasks> lt;
  // layout
  DevBuf<int> vertex_of, row_of, deg, xsrc, isrc, depth_ptr;
  DevBuf<std::uint8_t> loop, rowkind;
  DevBuf<long long> xptr, iptr;
  // tasks
  DevBuf<CacTask> cac;
  DevBuf<SccTask> small, small_big, lcta;
  DevBuf<LevelTask> ltasks;
  DevBuf<GridUnitState> gstate;
  DevBuf<SpmvBlock> blocks;
  DevBuf<unsigned short> meta;  // k_spmv_seg lane metadata, 32 per task
  DevBuf<HeavyRow> heavy;
  DevBuf<double> heavy_part;
  DevBuf<int> heavy_cnt;
  DevBuf<CrossTask> xheavy;
  DevBuf<double> xparts;
  DevBuf<int> xcnts;
  std::vector<CacSlice> cac_slices;
  DevBuf<double> small_scratch;
  int small_scratch_ld = 0;
  // work
  DevBuf<double> w, rank, s0, s1, pf, r3, r1, partial, total;
  DevBuf<SolveParams> params;
  DevBuf<DevStatus> status;
  DevBuf<long long> unit_iters;
  SolveParams* h_params = nullptr;
  DevStatus* h_status = nullptr;
  int nparts = 0;
  std::vector<long long> gu_rows, gu_nnz;   // per grid unit
  std::vector<cudaEvent_t> lev;              // per-launch event pairs (grid SpMV)
  int64_t launches = 0;
  int64_t spmv_launches = 0;
  // multi-GPU: grid SccLarge units row-sharded over `world` ranks of `comm`
  int shard = 0, nshards = 1;  // this process's rank / world size
  ncclComm_t comm = nullptr;
  std::vector<std::vector<int>> gu_bounds;  // per grid unit: world + 1 row bounds
  // exchange chunks: per grid unit, world * xchunks + 1 row bounds (rank r's
  // chunk j = [cuts[r * xchunks + j], cuts[r * xchunks + j + 1])), identical on
  // every rank; a chunk's s' rows are broadcast while the next chunk computes
  int xchunks = 1;
  std::vector<std::vector<int>> gu_cuts;
  bool dist_any = false;                     // some level's CTA units are split over the ranks
  // LR_UNIT_TIMES=1 at upload: per-CTA device timestamps of every level task
  // and large CAC, mapped to units after each solve (UnitRecord::wall_ms)
  bool unit_times = false;
  DevBuf<long long> ut_tasks, ut_cacs;
  std::vector<int64_t> task_unit_ptr;        // level task -> units (CSR)
  std::vector<int32_t> task_units;
  std::vector<int32_t> cac_unit;             // CacTask -> unit
  std::vector<int32_t> level_of_unit;
  std::vector<double> grid_level_ms;         // per level: its grid SpMV time (last solve)
  std::vector<double> h_unit_ms;             // per unit: device span of its tasks (last solve)
  bool unit_ms_valid = false;
  std::vector<std::uint8_t> h_unit_kind;     // host copies for the report of a split solve
  std::vector<long long> h_unit_edges;
  cudaStream_t xstream = nullptr;            // NCCL exchange, concurrent with the SpMV chunks
  std::vector<cudaEvent_t> xev;              // chunk j computed (compute stream -> exchange stream)
  cudaEvent_t xdone = nullptr;               // iteration's exchange done (exchange -> compute stream)
  DevBuf<double> maxbuf;                     // per grid unit: shard max, all-reduced
  DevBuf<double> cacpv;                      // pushed terms of CACs swept by cac_sweep_compact (n, or empty)
  // K5 (k_spmv_blk): dest-blocked, source-sorted in-edges of large grid units
  struct BlkUnit {
    DevBuf<unsigned> esrc;
    DevBuf<unsigned short> edst;
    DevBuf<BlkPart> parts;
    DevBuf<double> yacc;
    DevBuf<int> bcnt;
    BlkUnitDev dev{};
    size_t bytes() const { return esrc.bytes() + edst.bytes() + parts.bytes() + yacc.bytes() + bcnt.bytes(); }
  };
  std::vector<std::unique_ptr<BlkUnit>> blk;

  DeviceLayout dl() const {
    DeviceLayout L;
    L.n = n;
    L.vertex_of = vertex_of.p;
    L.row_of = row_of.p;
    L.deg = deg.p;
    L.loop = loop.p;
    L.rowkind = rowkind.p;
    L.xptr = xptr.p;
    L.xsrc = xsrc.p;
    L.iptr = iptr.p;
    L.isrc = isrc.p;
    return L;
  }
  ~lr_ctx() {
    if (device >= 0) cudaSetDevice(device);
    drop_graphs();
    for (cudaEvent_t e : xev) cudaEventDestroy(e);
    if (xdone) cudaEventDestroy(xdone);
    if (xstream) cudaStreamDestroy(xstream);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : lev)
      if (e) cudaEventDestroy(e);
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (join_ev) cudaEventDestroy(join_ev);
    if (pre_fork) cudaEventDestroy(pre_fork);
    if (pre_done) cudaEventDestroy(pre_done);
    if (pre) cudaStreamDestroy(pre);
    if (side) cudaStreamDestroy(side);
    if (stream) cudaStreamDestroy(stream);
    if (h_params) cudaFreeHost(h_params);
    if (h_status) cudaFreeHost(h_status);
    if (comm) nccl().comm_destroy(comm);
  }
};

static bool LR_NO_PREGATHER() {  // A/B switch: LR_PREGATHER=0 keeps the start weights inside k_cac_big
  const char* e = std::getenv("LR_PREGATHER");
  return e && std::atoi(e) == 0;
}

// In-edge order of a CTA power-series unit run by lcta_solve_staged's register
// rows: lane l of a warp loads the q-th in-edge of its row in the warp's q-th
// gather, one shared-memory load of a double per lane, so a gather costs as many
// wavefronts as its busiest bank pair (16 doubles span the 32 banks).  Per 16
// consecutive rows (a half-warp of one row set) and slot q < kLctaRegIdx, rows
// with the fewest remaining in-edges pick first, each the in-edge whose bank pair
// is least loaded in that slot; the rest keep their order.  The rows' sums are
// pairwise (order-insensitive up to rounding), so only the gathers' bank
// spread changes.  LR_BANK_ORDER=0 keeps the layout's order.
static bool bank_order_off() {
  const char* e = std::getenv("LR_BANK_ORDER");
  return e && std::atoi(e) == 0;
}

static void bank_balanced_order(const int64_t* iptr, const int* isrc, int rb, int re, std::vector<int>& out) {
  const int64_t eb = iptr[rb];
  out.assign(isrc + eb, isrc + iptr[re]);
  const int m = re - rb;
  std::vector<int> rem[16];
  for (int base = 0; base < m; base += 16) {
    const int nr = std::min(16, m - base);
    for (int l = 0; l < nr; ++l) {
      const int r = rb + base + l;
      const int64_t d = iptr[r + 1] - iptr[r];
      rem[l].clear();
      if (d > kCrossLight) continue;  // warp rows: not in registers
      rem[l].assign(isrc + iptr[r], isrc + iptr[r + 1]);
    }
    std::vector<int> pos(static_cast<size_t>(nr), 0), order(static_cast<size_t>(nr));
    for (int q = 0; q < kLctaRegIdx; ++q) {
      int load[16] = {};
      for (int l = 0; l < nr; ++l)  // rows without an in-edge for slot q read the zero slot (row m)
        if (rem[l].empty()) load[m & 15] = 1;
      for (int l = 0; l < nr; ++l) order[static_cast<size_t>(l)] = l;
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return rem[a].size() < rem[b].size(); });
      for (int l : order) {
        std::vector<int>& v = rem[l];
        if (v.empty()) continue;
        size_t best = 0;
        for (size_t k = 1; k < v.size() && load[(v[best] - rb) & 15] > 0; ++k)
          if (load[(v[k] - rb) & 15] < load[(v[best] - rb) & 15]) best = k;
        ++load[(v[best] - rb) & 15];
        const int r = rb + base + l;
        out[static_cast<size_t>(iptr[r] - eb + q)] = v[best];
        v.erase(v.begin() + static_cast<std::ptrdiff_t>(best));
        ++pos[static_cast<size_t>(l)];
      }
    }
    for (int l = 0; l < nr; ++l) {  // the tail (rows above kLctaRegIdx in-edges) in the layout's order
      const int r = rb + base + l;
      for (size_t k = 0; k < rem[l].size(); ++k)
        out[static_cast<size_t>(iptr[r] - eb + pos[static_cast<size_t>(l)] + static_cast<int64_t>(k))] = rem[l][k];
    }
  }
}

extern "C" {

lr_status lr_ctx_create(int device, lr_ctx** out) {
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    lrerr::set("no CUDA device available (the levelrank-b200 solve has no CPU fallback)");
    return LR_ECUDA;
  }
  if (device < 0 || device >= count) {
    lrerr::set("CUDA device index out of range");
    return LR_EINVAL;
  }
  auto* ctx = new lr_ctx;
  ctx->device = device;
  auto fail = [&](lr_status s) {
    delete ctx;
    return s;
  };
  if (cudaSetDevice(device) != cudaSuccess) {
    lrerr::set("cudaSetDevice failed");
    return fail(LR_ECUDA);
  }
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10) {
    lrerr::set(std::string("levelrank-b200 is built for sm_100a; found ") + prop.name);
    return fail(LR_ECUDA);
  }
  if (const cudaError_t e = configure_level_kernel(); e != cudaSuccess) {
    lrerr::set(std::string("level kernel setup failed: ") + cudaGetErrorString(e));
    return fail(LR_ECUDA);
  }
  if (const cudaError_t e = configure_kernels(); e != cudaSuccess) {
    lrerr::set(std::string("kernel setup failed: ") + cudaGetErrorString(e));
    return fail(LR_ECUDA);
  }
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    lrerr::set("CUDA stream creation failed");
    return fail(LR_ECUDA);
  }
  for (auto& e : ctx->ev)
    if (cudaEventCreate(&e) != cudaSuccess) {
      lrerr::set("cudaEventCreate failed");
      return fail(LR_ECUDA);
    }
  // the side stream outranks the main one, so a large CAC's 1024-thread CTA is
  // placed before the level's many k_level CTAs fill the SMs (otherwise it
  // waits for them and the level is serialised again)
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->pre, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->pre_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->pre_done, cudaEventDisableTiming) != cudaSuccess) {
    lrerr::set("CUDA side stream creation failed");
    return fail(LR_ECUDA);
  }
  if (cudaMallocHost(&ctx->h_params, sizeof(SolveParams)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_status, sizeof(DevStatus)) != cudaSuccess ||
      ctx->params.alloc(1) != cudaSuccess || ctx->status.alloc(1) != cudaSuccess) {
    lrerr::set("CUDA allocation failed");
    return fail(LR_ENOMEM);
  }
  *out = ctx;
  return LR_OK;
}

void lr_ctx_free(lr_ctx* ctx) { delete ctx; }

int32_t lr_ctx_blk_units(const lr_ctx* ctx) { return ctx ? static_cast<int32_t>(ctx->blk.size()) : 0; }

void* lr_ctx_stream(lr_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int64_t lr_ctx_device_bytes(const lr_ctx* c) {
  if (!c) return 0;
  return static_cast<int64_t>(c->vertex_of.bytes() + c->row_of.bytes() + c->deg.bytes() + c->xsrc.bytes() +
                              c->isrc.bytes() + c->depth_ptr.bytes() + c->loop.bytes() + c->rowkind.bytes() +
                              c->xptr.bytes() + c->iptr.bytes() + c->cac.bytes() + c->small.bytes() +
                              c->lcta.bytes() + c->gstate.bytes() + c->blocks.bytes() + c->meta.bytes() + c->heavy.bytes() +
                              c->heavy_part.bytes() + c->heavy_cnt.bytes() + c->small_scratch.bytes() +
                              c->w.bytes() + c->rank.bytes() + c->s0.bytes() + c->s1.bytes() + c->pf.bytes() +
                              c->r3.bytes() + c->r1.bytes() + c->partial.bytes() + c->unit_iters.bytes() +
                              [c] {
                                size_t b = 0;
                                for (const auto& u : c->blk) b += u->bytes();
                                return b;
                              }());
}

}  // extern "C"

// K5 for every level whose grid SpMV is one large unit on one GPU: its in-edges
// by dest-row blocks of BR rows, sorted by source (built on the device from the
// uploaded CSR, spmv.cu k_spmv_blk).  LR_BLK=0 keeps K4c everywhere;
// LR_BLK_MIN_ROWS (default 2^21) and LR_BLK_MIN_DEG (in-edges per row, default
// 8) set "large", LR_BLK_ROWS the block rows
// (default 16384), LR_BLK_PART the slots per part (default: about three parts
// per SM -- a block that is not split adds nothing to global memory; measured
// 5,238 / 5,365 / 5,422 / 5,421 GB/s at 8 / 4 / 2.7 / 1 parts per SM), LR_BLK_WIN the bank-balance window (0 or LR_BLK_BANKS=0: none),
// LR_BLK_SLACK the rows of entries per empty row (0: none).
static lr_status build_blk_units(lr_ctx* ctx, const lr_layout* L, const std::vector<GridUnitState>& gstate,
                                 cudaStream_t s) {
  ctx->blk.clear();
  auto env_int = [](const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
  };
  const char* e_on = std::getenv("LR_BLK");
  if ((e_on && std::atoi(e_on) == 0) || !spmv_seg()) return LR_OK;
  const char* e_min = std::getenv("LR_BLK_MIN_ROWS");
  const long long min_rows = e_min ? std::atoll(e_min) : (1ll << 21);
  const char* e_br = std::getenv("LR_BLK_ROWS");
  const int BR = std::max(32, std::min(e_br ? std::atoi(e_br) : 16384, (kMaxDynSmem / 8) - 64));
  int sms = 0;
  LR_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  // slots of a block's run: its entries in rows of 32 (one K5 gather
  // instruction), one empty row after every `slack` rows (free slots for the
  // bank balance), padded to whole chunks
  const int slack = std::max(0, env_int("LR_BLK_SLACK", kBlkSlack));
  int win = env_int("LR_BLK_BANKS", 1) == 0 ? 0 : env_int("LR_BLK_WIN", kBlkWindow);
  if (win != 0 && win != 256 && win != 1024 && win != 2048 && win != 4096 && win != 8192) win = kBlkWindow;
  // the layout of dest rows [row0, row0 + R) of the unit [u0, u0 + UR): its index
  // in ctx->blk, or -1 when the device has no room for it (the layout and its
  // build -- sort keys, double buffers: ~20 B per in-edge of scratch -- may not
  // fit next to a graph close to the HBM capacity: those rows keep K4c, which
  // needs nothing beyond the CSR)
  auto build_rows = [&](int u0, int UR, int row0, int R, int& index) -> lr_status {
    index = -1;
    const long long e_begin = L->iptr[row0], E = L->iptr[row0 + R] - e_begin;
    const int nb = static_cast<int>((static_cast<long long>(R) + BR - 1) / BR);
    std::vector<long long> pad_off(static_cast<size_t>(nb) + 1, 0);
    for (int b = 0; b < nb; ++b) {
      const long long cnt = L->iptr[row0 + std::min(R, (b + 1) * BR)] - L->iptr[row0 + b * BR];
      long long rows = (cnt + 31) / 32;
      if (slack > 0 && rows > 0) rows += (rows - 1) / slack;
      const long long slots = rows * 32;
      pad_off[static_cast<size_t>(b) + 1] = pad_off[static_cast<size_t>(b)] + (slots + kBlkChunk - 1) / kBlkChunk * kBlkChunk;
    }
    const long long total = pad_off.back();
    const char* e_part = std::getenv("LR_BLK_PART");
    long long P = e_part ? std::atoll(e_part) : total * 10 / (27ll * sms);
    P = std::max<long long>(kBlkChunk, (P + kBlkChunk - 1) / kBlkChunk * kBlkChunk);
    P = std::min<long long>(P, 1ll << 30);
    std::vector<BlkPart> parts;
    int nslots = 0;
    for (int b = 0; b < nb; ++b) {
      const long long a = pad_off[static_cast<size_t>(b)], n = pad_off[static_cast<size_t>(b) + 1] - a;
      const int np = static_cast<int>(std::max<long long>(1, (n + P - 1) / P));
      const int slot = np > 1 ? nslots++ : -1;
      for (int q = 0; q < np; ++q) {
        const long long lo = a + static_cast<long long>(q) * P, hi = std::min(a + n, lo + P);
        parts.push_back(BlkPart{lo, static_cast<int>(hi - lo), b, slot, np});
      }
    }
    // heaviest parts first: the launch's tail is made of the light ones
    std::stable_sort(parts.begin(), parts.end(), [](const BlkPart& x, const BlkPart& y) { return x.n > y.n; });
    auto U = std::make_unique<lr_ctx::BlkUnit>();
    auto build = [&]() -> cudaError_t {
      cudaError_t e;
      if ((e = U->esrc.alloc(static_cast<size_t>(total))) != cudaSuccess) return e;
      if ((e = U->edst.alloc(static_cast<size_t>(total))) != cudaSuccess) return e;
      if ((e = U->parts.upload(parts.data(), parts.size(), s)) != cudaSuccess) return e;
      if ((e = U->yacc.alloc(static_cast<size_t>(nslots) * BR)) != cudaSuccess) return e;
      if ((e = U->bcnt.alloc(static_cast<size_t>(nslots))) != cudaSuccess) return e;
      if ((e = cudaMemsetAsync(U->yacc.p, 0, U->yacc.bytes(), s)) != cudaSuccess) return e;
      if ((e = cudaMemsetAsync(U->bcnt.p, 0, U->bcnt.bytes(), s)) != cudaSuccess) return e;
      return build_blk_entries(ctx->iptr.p, ctx->isrc.p, e_begin, E, u0, UR, row0, R, BR, pad_off, slack, win,
                               U->esrc.p, U->edst.p, s);
    };
    if (const cudaError_t e = build(); e == cudaErrorMemoryAllocation) {
      cudaGetLastError();  // cleared: not sticky
      cudaStreamSynchronize(s);
      return LR_OK;
    } else {
      LR_CUDA_TRY(e);
    }
    U->dev = BlkUnitDev{U->esrc.p, U->edst.p, U->parts.p, static_cast<int>(parts.size()), u0, UR, row0, R, BR,
                        U->yacc.p, U->bcnt.p};
    index = static_cast<int>(ctx->blk.size());
    ctx->blk.push_back(std::move(U));
    return LR_OK;
  };
  for (LevelTasks& T : ctx->lt) {
    T.blk = -1;
    T.blk_chunks.clear();
    if (T.gu1 - T.gu0 != 1) continue;
    const int u = gstate[static_cast<size_t>(T.gu0)].unit;
    const int u0 = L->unit_row_begin[u], R = L->unit_row_begin[u + 1] - u0;
    if (R < min_rows || R <= 0) continue;
    const long long E = L->iptr[u0 + R] - L->iptr[u0];
    // sparse units (config 3's whole-graph baseline: 5.6 in-edges per row) have too
    // few entries per block for the sorted gathers to share lines: K4c
    if (E < static_cast<long long>(env_int("LR_BLK_MIN_DEG", 8)) * R) continue;
    bool any = false;
    if (!ctx->comm) {
      if (const lr_status bs = build_rows(u0, R, u0, R, T.blk); bs != LR_OK) return bs;
      any = T.blk >= 0;
    } else {
      // row-sharded: one layout per exchange chunk of this rank's shard (a chunk is
      // one launch, so that its s' rows can travel while the next chunk computes)
      const std::vector<int>& cuts = ctx->gu_cuts[static_cast<size_t>(T.gu0)];
      for (int xc = 0; xc < ctx->xchunks; ++xc) {
        const int c0 = cuts[static_cast<size_t>(ctx->shard * ctx->xchunks + xc)];
        const int c1 = cuts[static_cast<size_t>(ctx->shard * ctx->xchunks + xc) + 1];
        int idx = -1;
        if (c1 > c0)
          if (const lr_status bs = build_rows(u0, R, c0, c1 - c0, idx); bs != LR_OK) return bs;
        T.blk_chunks.push_back(idx);
        any = any || idx >= 0;
      }
    }
    // K5 streams its indices evict-first and gathers the pushed vector block after
    // block: a larger evict-last window than K4c's pays (measured at config 5:
    // 0 / 0.3 / 0.6 / 0.85 / 1.0 / 1.3 / 1.6 / 2.0 / 3.0 of L2 -> 4311 / 4978 /
    // 5276 / 5419 / 5451 / 5472 / 5484 / 5479 / 5462 GB/s)
    if (any && std::getenv("LR_L2_HOT_FRAC") == nullptr) {
      int l2 = 0;
      cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device);
      T.hot_rows = std::min<long long>(T.unit_rows, static_cast<long long>(1.6 * l2 / 16.0));
    }
  }
  return LR_OK;
}

extern "C" {

lr_status lr_ctx_upload(lr_ctx* ctx, const lr_layout* L) {
  if (!ctx || !L) {
    lrerr::set("null context or layout");
    return LR_EINVAL;
  }
  LR_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const int n = L->n;
  ctx->loaded = false;
  ctx->drop_graphs();
  ctx->n = n;
  ctx->n_levels = L->n_levels;
  ctx->n_units = L->n_units;
  const size_t nn = static_cast<size_t>(n);

  // per-row kind
  std::vector<std::uint8_t> rowkind(nn, kSingle);
  std::vector<CacTask> cac_w, cac_b;
  std::vector<SccTask> small, lcta;
  std::vector<GridUnitState> gstate;
  std::vector<SpmvBlock> blocks;
  std::vector<HeavyRow> heavy;
  std::vector<CrossTask> xheavy;
  std::vector<SccTask> small_big;
  std::vector<std::vector<std::pair<int, int>>> rowranges(static_cast<size_t>(L->n_levels));  // row tasks per level
  long long xparts = 0;
  int n_xslots = 0;
  long long heavy_parts = 0;
  ctx->lt.assign(static_cast<size_t>(L->n_levels), LevelTasks{});
  ctx->gu_rows.clear();
  ctx->gu_nnz.clear();
  ctx->gu_bounds.clear();
  ctx->gu_cuts.clear();
  ctx->xchunks = 1;
  if (ctx->comm) {
    const char* e = std::getenv("LR_XCHG_CHUNKS");
    ctx->xchunks = std::max(1, std::min(64, e ? std::atoi(e) : 4));
  }
  ctx->cac_slices.clear();
  // multi-GPU: the CTA-solved units of large levels split over the ranks
  // (LR_DIST_LEVELS=0 replicates them; LR_DIST_MIN_ROWS sets "large")
  ctx->dist_any = false;
  const bool dist_on = ctx->comm && [] {
    const char* e = std::getenv("LR_DIST_LEVELS");
    return !(e && std::atoi(e) == 0);
  }();
  const long long dist_min_rows = [] {
    const char* e = std::getenv("LR_DIST_MIN_ROWS");
    return e ? std::atoll(e) : (1ll << 16);
  }();
  ctx->h_unit_kind.assign(L->unit_kind, L->unit_kind + L->n_units);
  ctx->h_unit_edges.assign(L->unit_edges, L->unit_edges + L->n_units);
  int max_small = 0;
  bool small_needs_scratch = false;
  for (int li = 0; li < L->n_levels; ++li) {
    LevelTasks& T = ctx->lt[static_cast<size_t>(li)];
    T.rb = L->level_row_begin[li];
    T.re = L->level_row_begin[li + 1];
    std::vector<CacTask> lw, lm, lb;
    T.sl0 = static_cast<int>(ctx->cac_slices.size());
    T.xh0 = static_cast<int>(xheavy.size());
    for (int r = T.rb; r < T.re; ++r) {
      const long long xd = L->xptr[r + 1] - L->xptr[r];
      if (xd <= kCrossSplit) continue;
      const int nseg = static_cast<int>((xd + kCrossSeg - 1) / kCrossSeg);
      const int slot = n_xslots++;
      for (int sg = 0; sg < nseg; ++sg) {
        const long long e0 = L->xptr[r] + static_cast<long long>(sg) * kCrossSeg;
        xheavy.push_back(CrossTask{e0, xparts, static_cast<int>(std::min<long long>(kCrossSeg, L->xptr[r + 1] - e0)),
                                   r, sg, nseg, slot, 0});
      }
      xparts += nseg;
    }
    T.xh1 = static_cast<int>(xheavy.size());
    T.sm0 = static_cast<int>(small.size());
    T.sb0 = static_cast<int>(small_big.size());
    T.lc0 = static_cast<int>(lcta.size());
    T.gu0 = static_cast<int>(gstate.size());
    T.bk0 = static_cast<int>(blocks.size());
    std::vector<int> pending_chunks;  // exchange chunks of the level's (last) grid unit
    // this rank's rows of the level's CTA-solved units
    int my0 = T.rb, my1 = T.re;
    if (dist_on && T.re - T.rb >= dist_min_rows) {
      T.dist_bounds = split_level_rows(L->iptr, L->xptr, L->unit_row_begin, L->unit_kind, L->level_unit_begin[li],
                                       L->level_unit_begin[li + 1], ctx->nshards);
      my0 = T.dist_bounds[static_cast<size_t>(ctx->shard)];
      my1 = T.dist_bounds[static_cast<size_t>(ctx->shard) + 1];
      ctx->dist_any = true;
    }
    auto mine = [&](int a) { return a >= my0 && a < my1; };  // a whole unit starting at row a
    auto clip = [&](int a, int e) {  // this rank's part of a row-divisible range
      const int c0 = std::max(a, my0), c1 = std::min(e, my1);
      if (c1 > c0) rowranges[static_cast<size_t>(li)].emplace_back(c0, c1);
    };
    for (int u = L->level_unit_begin[li]; u < L->level_unit_begin[li + 1]; ++u) {
      const int rb = L->unit_row_begin[u], re = L->unit_row_begin[u + 1];
      const int m = re - rb;
      const std::uint8_t kind = L->unit_kind[u];
      std::uint8_t rk = kSingle;
      if (kind == 1) {
        rk = kCac;
        const long long db = L->cac_depth_begin[u];
        int nd = 0;
        while (L->depth_ptr[db + nd] < re) ++nd;  // depth_ptr[db+nd] == re ends the unit
        if (m > kCacBlockMaxRows) {
          // very large CAC: start weights by row tasks, then one grid-wide
          // launch per depth slice
          rowranges[static_cast<size_t>(li)].emplace_back(rb, re);
          for (int d = 0; d < nd; ++d) {
            const int r0 = L->depth_ptr[db + d], r1 = L->depth_ptr[db + d + 1];
            const int h0 = static_cast<int>(xheavy.size());
            for (int r = r0; r < r1; ++r) {
              const long long id = L->iptr[r + 1] - L->iptr[r];
              if (id <= kCrossLight) continue;
              const int nseg = static_cast<int>((id + kCrossSeg - 1) / kCrossSeg);
              const int slot = n_xslots++;
              for (int sg = 0; sg < nseg; ++sg) {
                const long long e0 = L->iptr[r] + static_cast<long long>(sg) * kCrossSeg;
                xheavy.push_back(CrossTask{e0, xparts, static_cast<int>(std::min<long long>(kCrossSeg, L->iptr[r + 1] - e0)),
                                           r, sg, nseg, slot, 0});
              }
              xparts += nseg;
            }
            ctx->cac_slices.push_back(CacSlice{r0, r1, h0, static_cast<int>(xheavy.size())});
          }
        } else {
          // (large CACs gather their own start weights in k_cac_big)
          if (m > kCacMidMaxRows) lb.push_back(CacTask{rb, re, db, nd, 0});  // side stream: every rank
          else if (mine(rb)) (m > kCacWarpMaxRows ? lm : lw).push_back(CacTask{rb, re, db, nd, 0});
        }
      } else if (kind == 2) {
        rk = kSmall;
        const long long ne = L->iptr[re] - L->iptr[rb];
        // dense units (in-edge stash) can outgrow k_level's shared memory at any
        // m: those go to the global-scratch kernel like the large ones
        if (m <= kSmallSmemMaxM && small_unit_smem_bytes(m, ne) <= kSmallSmemCap &&
            static_cast<size_t>(m + 1) * static_cast<size_t>(m + 2) * sizeof(double) <= kSmallSmemCap) {
          if (mine(rb)) small.push_back(SccTask{rb, re, u, 0, L->unit_edges[u]});
          T.sm_tile = std::max(T.sm_tile, small_unit_smem_bytes(m, ne));
          T.sm_max = std::max(T.sm_max, m);
        } else {  // beyond shared memory: global-scratch kernel after the level kernel
          small_big.push_back(SccTask{rb, re, u, 0, L->unit_edges[u]});
          rowranges[static_cast<size_t>(li)].emplace_back(rb, re);
          T.sb_max = std::max(T.sb_max, m);
          max_small = std::max(max_small, m);
          small_needs_scratch = true;
        }
      } else if (kind == 3) {
        const long long nnz = L->iptr[re] - L->iptr[rb];
        if (m <= kCtaLargeMaxRows && nnz <= kCtaLargeMaxNnz) {
          rk = kLargeCta;
          int has_heavy = 0;
          for (int r = rb; r < re && !has_heavy; ++r) has_heavy = L->iptr[r + 1] - L->iptr[r] > kCrossLight;
          if (mine(rb)) lcta.push_back(SccTask{rb, re, u, has_heavy, L->unit_edges[u]});
          // a multiple of 16 doubles (the 32 banks) above m: same bank map for
          // both pushed vectors, and room for the register path's zero slot
          T.lc_max = std::max(T.lc_max, (m + 2 + 15) & ~15);
        } else {
          rk = kLargeGrid;
          clip(rb, re);  // start values s0 = pf * w of the rows (exchanged after the level)
          const int gu = static_cast<int>(gstate.size());
          const size_t first_block = blocks.size();
          // multi-GPU: this rank owns rows [own0, own1) of the unit (nnz-balanced)
          ctx->gu_bounds.push_back(shard_bounds(L->iptr, rb, re, ctx->nshards));
          const int own0 = ctx->gu_bounds.back()[static_cast<size_t>(ctx->shard)];
          const int own1 = ctx->gu_bounds.back()[static_cast<size_t>(ctx->shard) + 1];
          // exchange chunks of every rank's shard (nnz-balanced, whole rows)
          ctx->gu_cuts.push_back(exchange_cuts(L->iptr, rb, re, ctx->nshards, ctx->xchunks));
          const std::vector<int>& my_cuts = ctx->gu_cuts.back();
          std::vector<int> chunk_bk;
          // K4c chunks hold <= kChunkNnz in-edges and never put an empty row
          // inside a multi-row tile (its row-start flag would collide)
          const int tile_nnz = spmv_seg() ? kChunkNnz : kTileNnz;
          const int seg_nnz = spmv_seg() ? kChunkSegNnz : kSegNnz;
          for (int xc = 0; xc < ctx->xchunks; ++xc) {
          const int cend = my_cuts[static_cast<size_t>(ctx->shard * ctx->xchunks + xc) + 1];
          chunk_bk.push_back(static_cast<int>(blocks.size()));
          int r = my_cuts[static_cast<size_t>(ctx->shard * ctx->xchunks + xc)];
          while (r < cend) {
            const long long len = L->iptr[r + 1] - L->iptr[r];
            if (len == 0 && spmv_seg()) {  // a run of rows without in-edges: y = 0
              const int start = r;
              while (r < cend && r - start < kTileRows && L->iptr[r + 1] == L->iptr[r]) ++r;
              blocks.push_back(SpmvBlock{L->iptr[start], 0, start, r, gu, -1, 0});
              continue;
            }
            if (len > tile_nnz) {
              if (len <= seg_nnz) {
                blocks.push_back(SpmvBlock{L->iptr[r], static_cast<int>(len), r, r + 1, gu, -1, 0});
              } else {
                const int nseg = static_cast<int>((len + seg_nnz - 1) / seg_nnz);
                const int hid = static_cast<int>(heavy.size());
                heavy.push_back(HeavyRow{r, nseg, heavy_parts});
                heavy_parts += nseg;
                for (int sg = 0; sg < nseg; ++sg) {
                  const long long nb = L->iptr[r] + static_cast<long long>(sg) * seg_nnz;
                  const int cnt = static_cast<int>(std::min<long long>(seg_nnz, L->iptr[r + 1] - nb));
                  blocks.push_back(SpmvBlock{nb, cnt, r, r + 1, gu, hid, sg});
                }
              }
              ++r;
              continue;
            }
            const int start = r;
            long long acc = 0;
            while (r < cend && r - start < kTileRows) {
              const long long l2 = L->iptr[r + 1] - L->iptr[r];
              if (l2 > tile_nnz || acc + l2 > tile_nnz || (l2 == 0 && spmv_seg())) break;
              acc += l2;
              ++r;
            }
            blocks.push_back(SpmvBlock{L->iptr[start], static_cast<int>(acc), start, r, gu, -1, 0});
          }
          }
          chunk_bk.push_back(static_cast<int>(blocks.size()));
          pending_chunks = std::move(chunk_bk);
          ctx->gu_rows.push_back(own1 - own0);  // roofline bookkeeping: this rank's share
          ctx->gu_nnz.push_back(L->iptr[own1] - L->iptr[own0]);
          GridUnitState g{};
          g.unit = u;
          g.nblocks = static_cast<int>(blocks.size() - first_block);
          g.edges = L->unit_edges[u];
          gstate.push_back(g);
        }
      }
      if (kind == 0) clip(rb, re);
      for (int r = rb; r < re; ++r) rowkind[static_cast<size_t>(r)] = rk;
    }
    T.cac_w0 = static_cast<int>(cac_w.size());
    cac_w.insert(cac_w.end(), lw.begin(), lw.end());
    T.cac_w1 = static_cast<int>(cac_w.size());
    T.cac_m0 = static_cast<int>(cac_w.size());
    cac_w.insert(cac_w.end(), lm.begin(), lm.end());
    T.cac_m1 = static_cast<int>(cac_w.size());
    T.cac_b0 = static_cast<int>(cac_b.size());
    cac_b.insert(cac_b.end(), lb.begin(), lb.end());
    T.cac_b1 = static_cast<int>(cac_b.size());
    T.sl1 = static_cast<int>(ctx->cac_slices.size());
    T.sm1 = static_cast<int>(small.size());
    T.sb1 = static_cast<int>(small_big.size());
    T.lc1 = static_cast<int>(lcta.size());
    T.gu1 = static_cast<int>(gstate.size());
    T.bk1 = static_cast<int>(blocks.size());
    if (T.gu1 - T.gu0 == 1 && ctx->xchunks > 1)
      for (const int bi : pending_chunks) T.chunk_bk.push_back(bi - T.bk0);
    // Hot head of the level's largest grid unit: its rows are ordered by
    // descending in-unit out-degree, so the first rows are the most gathered.
    // The head of s_in (read) and of s_out (written, read next iteration)
    // share a fraction of L2 (LR_L2_HOT_FRAC, default 0.85).
    {
      int l2 = 0;
      cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device);
      double frac = 0.85;  // measured at config 5: 0.4 / 0.55 / 0.7 / 0.85 / 1.0 -> 2782 / 2916 / 2998 / 3016 / 2998 GB/s
      if (const char* e = std::getenv("LR_L2_HOT_FRAC")) frac = std::atof(e);
      long long best = -1;
      for (int gi = T.gu0; gi < T.gu1; ++gi) {
        if (ctx->gu_nnz[static_cast<size_t>(gi)] <= best) continue;
        best = ctx->gu_nnz[static_cast<size_t>(gi)];
        const int u = gstate[static_cast<size_t>(gi)].unit;
        T.hot_begin = L->unit_row_begin[u];
        T.unit_rows = L->unit_row_begin[u + 1] - L->unit_row_begin[u];
        T.hot_rows = std::min<long long>(T.unit_rows, static_cast<long long>(frac * l2 / 16.0));
      }
      // The whole level's SpMV working set -- in-edge indices and row offsets,
      // rank, pf and both pushed vectors -- stays L2-resident across iterations
      // when it fits in a fraction of L2 (config 2: 82 MB); streamed operands
      // are then kept (evict-last) instead of streamed through (evict-first).
      double ws = 0.0;
      for (int gi = T.gu0; gi < T.gu1; ++gi)
        ws += 4.0 * static_cast<double>(ctx->gu_nnz[static_cast<size_t>(gi)]) +
              40.0 * static_cast<double>(ctx->gu_rows[static_cast<size_t>(gi)]);
      T.keep_stream = ws <= 0.75 * l2 ? 2 : 0;
      if (const char* e = std::getenv("LR_SPMV_KEEP")) T.keep_stream = std::atoi(e);
    }
  }
  // warp tasks first, then CTA tasks, in one array
  const int nw = static_cast<int>(cac_w.size());
  for (auto& T : ctx->lt) {
    T.cac_b0 += nw;
    T.cac_b1 += nw;
  }
  cac_w.insert(cac_w.end(), cac_b.begin(), cac_b.end());

  // CTA tasks of the fused per-level kernel, level by level
  std::vector<LevelTask> ltasks;
  bool any_compact = false;  // some k_cac_big CAC sweeps with structure-only staging
  for (int li = 0; li < L->n_levels; ++li) {
    LevelTasks& T = ctx->lt[static_cast<size_t>(li)];
    T.lt0 = static_cast<int>(ltasks.size());
    for (const auto& [a, b] : rowranges[static_cast<size_t>(li)])
      for (int r = a; r < b; r += 256) ltasks.push_back(LevelTask{kTaskRows, r, std::min(b, r + 256), 0});
    for (int i = T.cac_w0; i < T.cac_w1; i += 8) ltasks.push_back(LevelTask{kTaskCacWarps, i, std::min(T.cac_w1, i + 8), 0});
    for (int i = T.cac_m0; i < T.cac_m1; ++i) ltasks.push_back(LevelTask{kTaskCacBlock, i, i + 1, 0});
    for (int i = T.sm0; i < T.sm1; ++i) ltasks.push_back(LevelTask{kTaskSmall, i, i + 1, 0});
    for (int i = T.lc0; i < T.lc1; ++i) ltasks.push_back(LevelTask{kTaskLcta, i, i + 1, 0});
    T.lt1 = static_cast<int>(ltasks.size());
    // a k_cac_big CAC would gather its start weights in 32-row rounds of one
    // CTA: row tasks over many CTAs do it first
    T.xb0 = T.lt1;
    for (int i = T.cac_b0; i < T.cac_b1; ++i) {
      CacTask& t = cac_w[static_cast<size_t>(i)];
      if (t.row_end - t.row_begin <= kCacPregatherRows || LR_NO_PREGATHER()) continue;
      t.pregathered = 1;
      for (int r = t.row_begin; r < t.row_end; r += 256)
        ltasks.push_back(LevelTask{kTaskRows, r, std::min(t.row_end, r + 256), 0});
    }
    T.xb1 = static_cast<int>(ltasks.size());
    const size_t ld = static_cast<size_t>(T.sm_max) + 1;
    T.smem = std::max(T.sm_max > 0 ? ld * (ld + 1) * sizeof(double) : 0,
                      static_cast<size_t>(3) * static_cast<size_t>(T.lc_max) * sizeof(double));
    // CAC depth sweeps run from shared memory when the CAC's ranks and
    // in-edges fit (k_level budget kLevelStageBytes so that the level's other
    // CTAs keep their occupancy; k_cac_big up to kStageMaxBytes).
    auto need = [&](const CacTask& t) {
      return (cac_stage_need(t.row_end - t.row_begin, L->iptr[t.row_end] - L->iptr[t.row_begin]) + 15) & ~size_t{15};
    };
    size_t warp_need = 0, mid_need = 0;
    for (int i = T.cac_w0; i < T.cac_w1; ++i) {
      const size_t b = need(cac_w[static_cast<size_t>(i)]);
      if (8 * b <= kLevelStageBytes) warp_need = std::max(warp_need, 8 * b);
    }
    for (int i = T.cac_m0; i < T.cac_m1; ++i) {
      const size_t b = need(cac_w[static_cast<size_t>(i)]);
      if (b <= kLevelStageBytes) mid_need = std::max(mid_need, b);
    }
    T.smem = std::max({T.smem, T.sm_tile, warp_need, mid_need});
    // warp-tiled start-weight gathers of the CTA-solved units (cross_rows_cta)
    if (T.cac_m1 > T.cac_m0 || T.sm1 > T.sm0 || T.lc1 > T.lc0) T.smem = std::max(T.smem, kRowTaskSmem);
    if (!rowranges[static_cast<size_t>(li)].empty()) T.smem = std::max(T.smem, kRowTaskSmem);  // tiled row gathers
    for (int i = T.lc0; i < T.lc1; ++i) {  // CTA power series staged in shared memory where it fits
      const SccTask& lt = lcta[static_cast<size_t>(i)];
      const size_t b = lcta_stage_bytes(T.lc_max, L->iptr[lt.row_end] - L->iptr[lt.row_begin]);
      if (b <= kLctaStageMaxBytes) T.smem = std::max(T.smem, b);
    }
    T.big_smem = 0;
    for (int i = T.cac_b0; i < T.cac_b1; ++i) {
      const CacTask& t = cac_w[static_cast<size_t>(i)];
      const size_t b = need(t);
      const long long m = t.row_end - t.row_begin;
      const size_t bc = (cac_compact_need(m, L->iptr[t.row_end] - L->iptr[t.row_begin]) + 15) & ~size_t{15};
      if (b <= kStageMaxBytes) {
        T.big_smem = std::max(T.big_smem, b);
      } else if (m < 65536 && bc <= kStageMaxBytes) {
        T.big_smem = std::max(T.big_smem, bc);
        any_compact = true;
      }
    }
    if (T.cac_b1 > T.cac_b0) T.big_smem = std::max(T.big_smem, kBigCrossSmem);  // warp-tiled start weights
  }

  LR_CUDA_TRY(ctx->vertex_of.upload(L->vertex_of, nn, s));
  LR_CUDA_TRY(ctx->row_of.upload(L->row_of, nn, s));
  LR_CUDA_TRY(ctx->deg.upload(L->deg, nn, s));
  LR_CUDA_TRY(ctx->loop.upload(L->loop, nn, s));
  LR_CUDA_TRY(ctx->rowkind.upload(rowkind.data(), nn, s));
  LR_CUDA_TRY(ctx->xptr.upload(reinterpret_cast<const long long*>(L->xptr), nn + 1, s));
  LR_CUDA_TRY(ctx->xsrc.upload(L->xsrc, static_cast<size_t>(L->nnz_cross), s));
  LR_CUDA_TRY(ctx->iptr.upload(reinterpret_cast<const long long*>(L->iptr), nn + 1, s));
  // padded: K4c's aligned 256-slot index windows may reach past the last in-edge
  LR_CUDA_TRY(ctx->isrc.upload_padded(L->isrc, static_cast<size_t>(L->nnz_intra), kIdxPad, s));
  if (!bank_order_off())
    for (const SccTask& t : lcta) {
      if (t.row_end - t.row_begin > kLctaRegRows) continue;
      std::vector<int> es;
      bank_balanced_order(L->iptr, L->isrc, t.row_begin, t.row_end, es);
      if (!es.empty())
        LR_CUDA_TRY(cudaMemcpyAsync(ctx->isrc.p + L->iptr[t.row_begin], es.data(), es.size() * sizeof(int),
                                    cudaMemcpyHostToDevice, s));
    }
  LR_CUDA_TRY(ctx->depth_ptr.upload(L->depth_ptr, static_cast<size_t>(L->depth_ptr_len), s));
  if (const lr_status bs = build_blk_units(ctx, L, gstate, s); bs != LR_OK) return bs;
  // Large CACs' start weights in two halves (config-4 shaped chains of narrow
  // levels): each row's cross list is ordered by source level, so the terms from
  // levels solved at least two levels earlier are a prefix -- summed while the
  // previous level solves (kTaskRowsPart on the pre stream), the rest added at
  // the row's own level (kTaskRowsFin): same order, same rounding, off the
  // side stream's critical path.  Both levels must be captured together (no
  // grid SpMV between them).  Measured at config 4: 31.2 ms without, 31.9 ms with (the
  // finish tasks' latency is the same as the full gather's); off by default,
  // LR_XSPLIT=1 enables it.
  {
    const char* e = std::getenv("LR_XSPLIT");
    const bool on = e && std::atoi(e) != 0;
    bool any = false;
    for (size_t li = 1; on && li < ctx->lt.size(); ++li) {
      LevelTasks& T = ctx->lt[li];
      LevelTasks& P = ctx->lt[li - 1];
      if (T.xb1 <= T.xb0 || T.gu1 > T.gu0 || P.gu1 > P.gu0) continue;
      P.pt0 = static_cast<int>(ltasks.size());
      for (int i = T.xb0; i < T.xb1; ++i) {
        LevelTask& t = ltasks[static_cast<size_t>(i)];
        t.type = kTaskRowsFin;
        t.split = P.rb;
        ltasks.push_back(LevelTask{kTaskRowsPart, t.a, t.b, P.rb});
      }
      P.pt1 = static_cast<int>(ltasks.size());
      T.xb_fin = true;
      any = true;
    }
    if (any) LR_CUDA_TRY(ctx->xpart.alloc(static_cast<size_t>(ctx->n)));
  }
  LR_CUDA_TRY(ctx->cac.upload(cac_w.data(), cac_w.size(), s));
  LR_CUDA_TRY(ctx->small.upload(small.data(), small.size(), s));
  LR_CUDA_TRY(ctx->small_big.upload(small_big.data(), small_big.size(), s));
  LR_CUDA_TRY(ctx->ltasks.upload(ltasks.data(), ltasks.size(), s));
  ctx->unit_times = [] {
    const char* e = std::getenv("LR_UNIT_TIMES");
    return e && std::atoi(e) != 0;
  }();
  ctx->unit_ms_valid = false;
  if (ctx->unit_times) {
    auto unit_of_row = [&](int r) {
      return static_cast<int32_t>(std::upper_bound(L->unit_row_begin, L->unit_row_begin + L->n_units + 1, r) -
                                  L->unit_row_begin - 1);
    };
    ctx->task_unit_ptr.assign(1, 0);
    ctx->task_units.clear();
    for (const LevelTask& t : ltasks) {
      switch (t.type) {
        case kTaskCacWarps:
          for (int i = t.a; i < t.b; ++i) ctx->task_units.push_back(unit_of_row(cac_w[static_cast<size_t>(i)].row_begin));
          break;
        case kTaskCacBlock:
          ctx->task_units.push_back(unit_of_row(cac_w[static_cast<size_t>(t.a)].row_begin));
          break;
        case kTaskSmall:
          ctx->task_units.push_back(small[static_cast<size_t>(t.a)].unit);
          break;
        case kTaskLcta:
          ctx->task_units.push_back(lcta[static_cast<size_t>(t.a)].unit);
          break;
        default:  // row tasks: rows of one unit
          ctx->task_units.push_back(unit_of_row(t.a));
          break;
      }
      ctx->task_unit_ptr.push_back(static_cast<int64_t>(ctx->task_units.size()));
    }
    ctx->cac_unit.resize(cac_w.size());
    for (size_t i = 0; i < cac_w.size(); ++i) ctx->cac_unit[i] = unit_of_row(cac_w[i].row_begin);
    ctx->level_of_unit.assign(static_cast<size_t>(L->n_units), 0);
    for (int li = 0; li < L->n_levels; ++li)
      for (int u = L->level_unit_begin[li]; u < L->level_unit_begin[li + 1]; ++u) ctx->level_of_unit[static_cast<size_t>(u)] = li;
    LR_CUDA_TRY(ctx->ut_tasks.alloc(3 * std::max<size_t>(ltasks.size(), 1)));
    LR_CUDA_TRY(ctx->ut_cacs.alloc(3 * std::max<size_t>(cac_w.size(), 1)));
  }
  LR_CUDA_TRY(ctx->lcta.upload(lcta.data(), lcta.size(), s));
  LR_CUDA_TRY(ctx->gstate.upload(gstate.data(), gstate.size(), s));
  LR_CUDA_TRY(ctx->blocks.upload(blocks.data(), blocks.size(), s));
  // k_spmv_seg tiles: per lane of the aligned 256-slot window, the row-start
  // flags of its 8 slots and the number of rows starting before them
  std::vector<unsigned short> meta;
  if (spmv_seg()) {
    meta.assign(blocks.size() * 32, 0);
    for (size_t t = 0; t < blocks.size(); ++t) {
      const SpmvBlock& b = blocks[t];
      if (b.heavy >= 0 || b.nnz > kChunkNnz || b.nnz == 0) continue;
      const long long A = b.nnz_begin & ~7ll;
      unsigned char fl[32] = {};
      for (int r = b.row_begin; r < b.row_end; ++r) {
        const int slot = static_cast<int>(L->iptr[r] - A);
        fl[slot >> 3] = static_cast<unsigned char>(fl[slot >> 3] | (1u << (slot & 7)));
      }
      int before = 0;
      for (int l = 0; l < 32; ++l) {
        meta[t * 32 + static_cast<size_t>(l)] = static_cast<unsigned short>(fl[l] | (before << 8));
        before += __builtin_popcount(fl[l]);
      }
    }
  }
  LR_CUDA_TRY(ctx->meta.upload(meta.data(), meta.size(), s));
  LR_CUDA_TRY(ctx->heavy.upload(heavy.data(), heavy.size(), s));
  LR_CUDA_TRY(ctx->heavy_part.alloc(static_cast<size_t>(heavy_parts)));
  LR_CUDA_TRY(ctx->heavy_cnt.alloc(heavy.size()));
  LR_CUDA_TRY(ctx->xheavy.upload(xheavy.data(), xheavy.size(), s));
  LR_CUDA_TRY(ctx->xparts.alloc(static_cast<size_t>(xparts)));
  LR_CUDA_TRY(ctx->xcnts.alloc(static_cast<size_t>(n_xslots)));
  LR_CUDA_TRY(cudaMemsetAsync(ctx->xcnts.p, 0, ctx->xcnts.bytes(), s));
  LR_CUDA_TRY(cudaMemsetAsync(ctx->heavy_cnt.p, 0, ctx->heavy_cnt.bytes(), s));
  ctx->small_scratch.reset();
  ctx->small_scratch_ld = max_small + 1;
  if (small_needs_scratch) {
    const size_t ld = static_cast<size_t>(max_small) + 1;
    LR_CUDA_TRY(ctx->small_scratch.alloc(static_cast<size_t>(kSmallScratchBlocks) * ld * (ld + 2)));
  }
  LR_CUDA_TRY(ctx->w.alloc(nn));
  LR_CUDA_TRY(ctx->rank.alloc(nn));
  LR_CUDA_TRY(ctx->pf.alloc(nn));
  LR_CUDA_TRY(ctx->r3.alloc(nn));
  LR_CUDA_TRY(ctx->r1.alloc(nn));
  const bool any_grid = !gstate.empty();
  LR_CUDA_TRY(ctx->s0.alloc(any_grid ? nn : 0));
  LR_CUDA_TRY(ctx->cacpv.alloc(any_compact ? nn : 0));
  LR_CUDA_TRY(ctx->s1.alloc(any_grid ? nn : 0));
  LR_CUDA_TRY(ctx->maxbuf.alloc(gstate.size()));
  ctx->nparts = static_cast<int>((nn + kOutBlock - 1) / kOutBlock);
  LR_CUDA_TRY(ctx->partial.alloc(static_cast<size_t>(std::max(ctx->nparts, 1))));
  LR_CUDA_TRY(ctx->total.alloc(1));
  LR_CUDA_TRY(ctx->unit_iters.alloc(static_cast<size_t>(L->n_units)));
  LR_CUDA_TRY(cudaStreamSynchronize(s));
  ctx->loaded = true;
  return LR_OK;
}

// Multi-GPU exchange for the grid units of one level: each rank's row shard of
// `buf` is broadcast in place to all ranks (grouped broadcasts = an all-gather
// with uneven shards); with_max also all-reduces the shard maxima in maxbuf.
static lr_status exchange_shards(lr_ctx* ctx, const LevelTasks& T, double* buf, bool with_max) {
  const NcclApi& nc = nccl();
  LR_NCCL_TRY(nc.group_start());
  for (int gi = T.gu0; gi < T.gu1; ++gi) {
    const std::vector<int>& b = ctx->gu_bounds[static_cast<size_t>(gi)];
    for (int r = 0; r < ctx->nshards; ++r) {
      const size_t cnt = static_cast<size_t>(b[static_cast<size_t>(r) + 1] - b[static_cast<size_t>(r)]);
      if (cnt == 0) continue;
      double* p = buf + b[static_cast<size_t>(r)];
      LR_NCCL_TRY(nc.broadcast(p, p, cnt, ncclDouble, r, ctx->comm, ctx->stream));
    }
  }
  if (with_max)
    LR_NCCL_TRY(nc.all_reduce(ctx->maxbuf.p + T.gu0, ctx->maxbuf.p + T.gu0, static_cast<size_t>(T.gu1 - T.gu0),
                              ncclDouble, ncclMax, ctx->comm, ctx->stream));
  LR_NCCL_TRY(nc.group_end());
  return LR_OK;
}

// One power-series iteration of a level's single grid unit, row-sharded over
// the ranks and cut into exchange chunks: SpMV chunk j on the compute stream,
// then on the exchange stream the broadcasts of every rank's chunk j of s'
// (and, after the last chunk, the all-reduce of the shard maxima) -- so the
// exchange of chunk j overlaps the SpMV of chunk j + 1.  The chunks' maxima
// accumulate in the unit state; only the last chunk publishes them.
static lr_status chunked_iteration(lr_ctx* ctx, const LevelTasks& T, const DeviceLayout& L, const double* sin,
                                   double* sout, int64_t& launches) {
  cudaStream_t s = ctx->stream;
  const int C = static_cast<int>(T.chunk_bk.size()) - 1;
  if (!ctx->xstream) LR_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->xstream, cudaStreamNonBlocking));
  if (!ctx->xdone) LR_CUDA_TRY(cudaEventCreateWithFlags(&ctx->xdone, cudaEventDisableTiming));
  while (static_cast<int>(ctx->xev.size()) < C) {
    cudaEvent_t e;
    LR_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->xev.push_back(e);
  }
  const NcclApi& nc = nccl();
  const std::vector<int>& cuts = ctx->gu_cuts[static_cast<size_t>(T.gu0)];
  for (int j = 0; j < C; ++j) {
    const int b0 = T.bk0 + T.chunk_bk[static_cast<size_t>(j)], b1 = T.bk0 + T.chunk_bk[static_cast<size_t>(j) + 1];
    if (static_cast<size_t>(j) < T.blk_chunks.size() && T.blk_chunks[static_cast<size_t>(j)] >= 0)
      launch_spmv_blk(ctx->blk[static_cast<size_t>(T.blk_chunks[static_cast<size_t>(j)])]->dev, T.gu0, ctx->gstate.p,
                      ctx->params.p, ctx->pf.p, ctx->rank.p, sin, sout, ctx->unit_iters.p, ctx->status.p, T.hot_begin,
                      T.hot_rows, T.unit_rows, s, ctx->maxbuf.p, j < C - 1 ? 1 : 0);
    else
      launch_grid_iter(L, ctx->blocks.p + b0, ctx->meta.p ? ctx->meta.p + static_cast<size_t>(b0) * 32 : nullptr, b1 - b0,
                       T.gu0, 1, ctx->gstate.p, ctx->heavy.p, ctx->heavy_part.p, ctx->heavy_cnt.p, ctx->params.p,
                       ctx->pf.p, ctx->rank.p, sin, sout, ctx->unit_iters.p, ctx->status.p, T.hot_begin, T.hot_rows,
                       T.unit_rows, T.keep_stream, ctx->maxbuf.p, s, j < C - 1 ? 1 : 0);
    ++launches;
    LR_CUDA_TRY(cudaEventRecord(ctx->xev[static_cast<size_t>(j)], s));
    LR_CUDA_TRY(cudaStreamWaitEvent(ctx->xstream, ctx->xev[static_cast<size_t>(j)], 0));
    LR_NCCL_TRY(nc.group_start());
    for (int q = 0; q < ctx->nshards; ++q) {
      const int r0 = cuts[static_cast<size_t>(q * C + j)], r1 = cuts[static_cast<size_t>(q * C + j) + 1];
      if (r1 > r0)
        LR_NCCL_TRY(nc.broadcast(sout + r0, sout + r0, static_cast<size_t>(r1 - r0), ncclDouble, q, ctx->comm,
                                 ctx->xstream));
    }
    if (j == C - 1)
      LR_NCCL_TRY(nc.all_reduce(ctx->maxbuf.p + T.gu0, ctx->maxbuf.p + T.gu0, 1, ncclDouble, ncclMax, ctx->comm,
                                ctx->xstream));
    LR_NCCL_TRY(nc.group_end());
  }
  LR_CUDA_TRY(cudaEventRecord(ctx->xdone, ctx->xstream));
  LR_CUDA_TRY(cudaStreamWaitEvent(s, ctx->xdone, 0));
  launch_grid_finish(ctx->gstate.p, T.gu0, 1, ctx->params.p, ctx->unit_iters.p, ctx->status.p, ctx->maxbuf.p, s);
  ++launches;
  return LR_OK;
}

// A level whose CTA-solved units are split over the ranks: each rank's row
// range (its units' ranks, and the start values s0 of grid rows) broadcast to
// every rank -- grouped in-place broadcasts, an all-gather with uneven parts.
// Rows in the range that every rank computed (large CACs, global-scratch small
// SCCs, CAC slices) carry the same values everywhere, so overwriting them is
// harmless.
static lr_status exchange_level(lr_ctx* ctx, const LevelTasks& T) {
  const NcclApi& nc = nccl();
  LR_NCCL_TRY(nc.group_start());
  for (int q = 0; q < ctx->nshards; ++q) {
    const int r0 = T.dist_bounds[static_cast<size_t>(q)], r1 = T.dist_bounds[static_cast<size_t>(q) + 1];
    if (r1 <= r0) continue;
    LR_NCCL_TRY(nc.broadcast(ctx->rank.p + r0, ctx->rank.p + r0, static_cast<size_t>(r1 - r0), ncclDouble, q,
                             ctx->comm, ctx->stream));
    if (T.gu1 > T.gu0)
      LR_NCCL_TRY(nc.broadcast(ctx->s0.p + r0, ctx->s0.p + r0, static_cast<size_t>(r1 - r0), ncclDouble, q, ctx->comm,
                               ctx->stream));
  }
  LR_NCCL_TRY(nc.group_end());
  return LR_OK;
}

static lr_status solve_on_device(lr_ctx* ctx, const double* w_dev, double c, double tol, double* r3_dev,
                                 double* r1_dev, lr_solve_info* info, int64_t* unit_iters) {
  const lr_status pv = lr_validate_params(c, tol);
  if (pv != LR_OK) return pv;
  if (!ctx || !ctx->loaded) {
    lrerr::set("context has no uploaded layout");
    return LR_EINVAL;
  }
  LR_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const DeviceLayout L = ctx->dl();
  ctx->h_params->c = c;
  ctx->h_params->tol = tol;
  ctx->h_params->cap = lr_iteration_cap(c, tol);
  int64_t launches = 0, spmv_launches = 0;
  float spmv_ms = 0.f;
  double active_ms = 0.0;
  int64_t active_launches = 0, spmv_bytes = 0, spmv_edges = 0;
  LR_CUDA_TRY(cudaMemcpyAsync(ctx->params.p, ctx->h_params, sizeof(SolveParams), cudaMemcpyHostToDevice, s));
  LR_CUDA_TRY(cudaMemsetAsync(ctx->status.p, 0, sizeof(DevStatus), s));
  if (ctx->n_units > 0) LR_CUDA_TRY(cudaMemsetAsync(ctx->unit_iters.p, 0, ctx->unit_iters.bytes(), s));
  if (ctx->unit_times) {
    LR_CUDA_TRY(cudaMemsetAsync(ctx->ut_tasks.p, 0, ctx->ut_tasks.bytes(), s));
    LR_CUDA_TRY(cudaMemsetAsync(ctx->ut_cacs.p, 0, ctx->ut_cacs.bytes(), s));
    ctx->grid_level_ms.assign(ctx->lt.size(), 0.0);
  }
  LR_CUDA_TRY(cudaEventRecord(ctx->ev[0], s));
  // LR_LEVEL_PROF=1: per-level timing of k_level's CTAs by task type (diagnostic, synchronises every level)
  const bool prof_on = std::getenv("LR_LEVEL_PROF") != nullptr;
  const bool prof_detail = prof_on && std::atoi(std::getenv("LR_LEVEL_PROF")) > 1;
  DevBuf<long long> prof_buf;
  double prof_max[5] = {0, 0, 0, 0, 0}, prof_crit[5] = {0, 0, 0, 0, 0}, prof_span = 0;
  long long prof_cnt[5] = {0, 0, 0, 0, 0};
  cudaEvent_t pev[3] = {nullptr, nullptr, nullptr};
  double side_main = 0, side_side = 0, side_crit = 0;
  long long side_longer = 0, side_levels = 0;
  if (prof_on)
    for (auto& e : pev) LR_CUDA_TRY(cudaEventCreate(&e));
  if (prof_on) {
    int most = 1;
    for (const LevelTasks& T : ctx->lt) most = std::max({most, T.lt1 - T.lt0, T.xb1 - T.xb0});
    LR_CUDA_TRY(prof_buf.alloc(static_cast<size_t>(3 * most)));
    LR_CUDA_TRY(set_level_prof(prof_buf.p));
  }
  // graph replays read the weights from ctx->w (a fixed address)
  const bool use_graphs = !prof_on && [] {
    const char* e = std::getenv("LR_GRAPHS");
    return !(e && std::atoi(e) == 0);
  }();
  if (use_graphs && w_dev != ctx->w.p && ctx->n > 0) {
    LR_CUDA_TRY(cudaMemcpyAsync(ctx->w.p, w_dev, static_cast<size_t>(ctx->n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    w_dev = ctx->w.p;
  }
  launch_prep(L, w_dev, ctx->params.p, ctx->pf.p, ctx->status.p, s);
  ++launches;
  // everything of one level that the host does not steer: enqueued directly, or
  // captured into a segment graph
  auto static_level = [&](const LevelTasks& T, int64_t& nl) -> lr_status {
    // the previous level's early partial sums of this level's large CACs
    if (T.xb_fin) LR_CUDA_TRY(cudaStreamWaitEvent(s, ctx->pre_done, 0));
    // early partial sums of the NEXT level's large CACs, concurrent with this level
    if (T.pt1 > T.pt0) {
      LR_CUDA_TRY(cudaEventRecord(ctx->pre_fork, s));
      LR_CUDA_TRY(cudaStreamWaitEvent(ctx->pre, ctx->pre_fork, 0));
      launch_level(L, ctx->ltasks.p + T.pt0, T.pt1 - T.pt0, ctx->cac.p, ctx->depth_ptr.p, ctx->small.p, ctx->lcta.p, 0,
                   0, kRowTaskSmem, w_dev, ctx->params.p, ctx->pf.p, ctx->rank.p, ctx->s0.p, ctx->unit_iters.p,
                   ctx->status.p, true, ctx->pre, /*profile=*/false, ctx->xpart.p,
                   ctx->unit_times ? ctx->ut_tasks.p + 3 * static_cast<size_t>(T.pt0) : nullptr);
      LR_CUDA_TRY(cudaEventRecord(ctx->pre_done, ctx->pre));
      ++nl;
    }
    // K1 for rows with more than kCrossSplit cross in-edges (split over warps)
    if (T.xh1 > T.xh0) {
      launch_cross_heavy(L, ctx->xheavy.p + T.xh0, T.xh1 - T.xh0, w_dev, ctx->params.p, ctx->pf.p, ctx->rank.p,
                         ctx->s0.p, ctx->xparts.p, ctx->xcnts.p, s);
      ++nl;
    }
    // large CACs (start weights + depth sweep, 1024-thread CTAs) on the side
    // stream, concurrently with the level's k_level: units of one level are
    // independent, both only read ranks of the levels above
    const bool fork = T.cac_b1 > T.cac_b0;
    if (prof_on && fork) LR_CUDA_TRY(cudaEventRecord(pev[0], s));
    if (fork) {
      LR_CUDA_TRY(cudaEventRecord(ctx->fork_ev, s));
      LR_CUDA_TRY(cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0));
      if (T.xb1 > T.xb0) {
        launch_level(L, ctx->ltasks.p + T.xb0, T.xb1 - T.xb0, ctx->cac.p, ctx->depth_ptr.p, ctx->small.p, ctx->lcta.p,
                     0, 0, kRowTaskSmem, w_dev, ctx->params.p, ctx->pf.p, ctx->rank.p, ctx->s0.p, ctx->unit_iters.p,
                     ctx->status.p, T.xb_fin, ctx->side, /*profile=*/false, ctx->xpart.p,
                     ctx->unit_times ? ctx->ut_tasks.p + 3 * static_cast<size_t>(T.xb0) : nullptr);
        ++nl;
      }
      launch_cac_big(L, ctx->cac.p + T.cac_b0, T.cac_b1 - T.cac_b0, ctx->depth_ptr.p, w_dev, ctx->params.p, ctx->pf.p,
                     ctx->rank.p, ctx->s0.p, ctx->cacpv.n ? ctx->cacpv.p : nullptr, T.big_smem, ctx->side,
                     ctx->unit_times ? ctx->ut_cacs.p + 3 * static_cast<size_t>(T.cac_b0) : nullptr);
      if (prof_on) LR_CUDA_TRY(cudaEventRecord(pev[2], ctx->side));
      LR_CUDA_TRY(cudaEventRecord(ctx->join_ev, ctx->side));
      ++nl;
    }
    // everything that fits a CTA: K1 + singletons + CACs + small SCCs + CTA-sized large SCCs
    if (T.lt1 > T.lt0) {
      launch_level(L, ctx->ltasks.p + T.lt0, T.lt1 - T.lt0, ctx->cac.p, ctx->depth_ptr.p, ctx->small.p, ctx->lcta.p,
                   T.sm_max + 1, T.lc_max, T.smem, w_dev, ctx->params.p, ctx->pf.p, ctx->rank.p, ctx->s0.p,
                   ctx->unit_iters.p, ctx->status.p, T.sm1 > T.sm0 || T.lc1 > T.lc0, s, true, nullptr,
                   ctx->unit_times ? ctx->ut_tasks.p + 3 * static_cast<size_t>(T.lt0) : nullptr);
      ++nl;
      if (prof_on && fork) LR_CUDA_TRY(cudaEventRecord(pev[1], s));
      if (prof_on) {  // LR_LEVEL_PROF: per task type, the longest CTA of this level
        const int nt = T.lt1 - T.lt0;
        std::vector<long long> h(static_cast<size_t>(3 * nt));
        LR_CUDA_TRY(cudaMemcpyAsync(h.data(), prof_buf.p, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, s));
        LR_CUDA_TRY(cudaStreamSynchronize(s));
        long long lo = h[1], hi = h[2];
        double mx[5] = {0, 0, 0, 0, 0};
        for (int i = 0; i < nt; ++i) {
          const int ty = static_cast<int>(h[3 * i]);
          lo = std::min(lo, h[3 * i + 1]);
          hi = std::max(hi, h[3 * i + 2]);
          mx[ty] = std::max(mx[ty], (h[3 * i + 2] - h[3 * i + 1]) * 1e-3);
          prof_cnt[ty] += 1;
        }
        prof_span += (hi - lo) * 1e-3;
        if (prof_detail)
          std::fprintf(stderr, "[LR_LEVEL_PROF] level ctas %d span %.1f us  max rows %.1f cacw %.1f cacb %.1f small %.1f lcta %.1f\n",
                       nt, (hi - lo) * 1e-3, mx[0], mx[1], mx[2], mx[3], mx[4]);
        int arg = 0;
        for (int ty = 0; ty < 5; ++ty) {
          prof_max[ty] += mx[ty];
          if (mx[ty] > mx[arg]) arg = ty;
        }
        prof_crit[arg] += mx[arg];
      }
    }
    if (fork) LR_CUDA_TRY(cudaStreamWaitEvent(s, ctx->join_ev, 0));
    if (prof_on && fork && T.lt1 > T.lt0) {  // main-stream level kernel vs the side stream's large CACs
      LR_CUDA_TRY(cudaStreamSynchronize(s));
      float mm = 0.f, ss = 0.f;
      cudaEventElapsedTime(&mm, pev[0], pev[1]);
      cudaEventElapsedTime(&ss, pev[0], pev[2]);
      side_main += mm;
      side_side += ss;
      side_crit += std::max(mm, ss);
      side_longer += ss > mm;
      ++side_levels;
    }
    if (T.sb1 > T.sb0) {
      launch_small(L, ctx->small_big.p + T.sb0, T.sb1 - T.sb0, ctx->small_scratch_ld - 1, ctx->pf.p, ctx->rank.p,
                   ctx->small_scratch.p, ctx->status.p, s);
      ++nl;
    }
    for (int i = T.sl0; i < T.sl1; ++i) {
      const CacSlice& sl = ctx->cac_slices[static_cast<size_t>(i)];
      launch_cac_slice(L, sl.r0, sl.r1, ctx->params.p, ctx->rank.p, s);
      ++nl;
      if (sl.h1 > sl.h0) {
        launch_cac_heavy(L, ctx->xheavy.p + sl.h0, sl.h1 - sl.h0, ctx->params.p, ctx->rank.p, ctx->xparts.p,
                         ctx->xcnts.p, s);
        ++nl;
      }
    }
    return LR_OK;
  };
  if (use_graphs && !ctx->segs_built) {
    // a level with a grid SpMV or with an exchange of split units is enqueued
    // directly every solve; runs of the others are captured
    auto capturable = [&](size_t q) { return ctx->lt[q].gu1 == ctx->lt[q].gu0 && ctx->lt[q].dist_bounds.empty(); };
    for (size_t li = 0; li < ctx->lt.size();) {
      if (!capturable(li)) {
        ++li;
        continue;
      }
      size_t lj = li;
      while (lj < ctx->lt.size() && capturable(lj)) ++lj;
      lr_ctx::Segment seg{static_cast<int>(li), static_cast<int>(lj), 0, nullptr};
      LR_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      lr_status cst = LR_OK;
      for (size_t q = li; q < lj && cst == LR_OK; ++q) cst = static_level(ctx->lt[q], seg.launches);
      cudaGraph_t graph = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(s, &graph);
      if (cst != LR_OK) return cst;
      LR_CUDA_TRY(ce);
      const cudaError_t ie = cudaGraphInstantiate(&seg.exec, graph, 0);
      cudaGraphDestroy(graph);
      LR_CUDA_TRY(ie);
      ctx->segs.push_back(seg);
      li = lj;
    }
    ctx->segs_built = true;
  }
  size_t next_seg = 0;
  for (size_t li = 0; li < ctx->lt.size(); ++li) {
    if (use_graphs && next_seg < ctx->segs.size() && static_cast<size_t>(ctx->segs[next_seg].begin) == li) {
      const lr_ctx::Segment& seg = ctx->segs[next_seg++];
      LR_CUDA_TRY(cudaGraphLaunch(seg.exec, s));
      launches += seg.launches;
      li = static_cast<size_t>(seg.end) - 1;
      continue;
    }
    const LevelTasks& T = ctx->lt[li];
    if (const lr_status ls = static_level(T, launches); ls != LR_OK) return ls;
    if (!T.dist_bounds.empty())  // every rank's rows of the split units to every rank
      if (const lr_status xs = exchange_level(ctx, T); xs != LR_OK) return xs;
    if (T.gu1 > T.gu0) {
      launch_grid_reset(ctx->gstate.p + T.gu0, T.gu1 - T.gu0, ctx->status.p, s);
      ++launches;
      LR_CUDA_TRY(cudaEventRecord(ctx->ev[2], s));
      long long k = 0;
      const long long cap = ctx->h_params->cap;
      int batch = 4;
      for (;;) {
        for (int j = 0; j < batch; ++j) {
          ++k;
          const double* sin = (k & 1) ? ctx->s0.p : ctx->s1.p;
          double* sout = (k & 1) ? ctx->s1.p : ctx->s0.p;
          // one event per launch (lev[k] after launch k, lev[0] before the
          // first): the active launches' time is lev[0] -> lev[last active]
          while (ctx->lev.size() < static_cast<size_t>(k + 1)) {
            cudaEvent_t e;
            LR_CUDA_TRY(cudaEventCreate(&e));
            ctx->lev.push_back(e);
          }
          if (k == 1) LR_CUDA_TRY(cudaEventRecord(ctx->lev[0], s));
          const bool sharded = ctx->comm != nullptr;
          if (sharded && T.chunk_bk.size() > 2) {  // exchange overlapped chunk by chunk
            if (const lr_status xs = chunked_iteration(ctx, T, L, sin, sout, launches); xs != LR_OK) return xs;
            LR_CUDA_TRY(cudaEventRecord(ctx->lev[static_cast<size_t>(k)], s));
            ++spmv_launches;
            continue;
          }
          if (T.blk >= 0 && !sharded) {
            launch_spmv_blk(ctx->blk[static_cast<size_t>(T.blk)]->dev, T.gu0, ctx->gstate.p, ctx->params.p, ctx->pf.p,
                            ctx->rank.p, sin, sout, ctx->unit_iters.p, ctx->status.p, T.hot_begin, T.hot_rows,
                            T.unit_rows, s);
            LR_CUDA_TRY(cudaEventRecord(ctx->lev[static_cast<size_t>(k)], s));
            ++launches;
            ++spmv_launches;
            continue;
          }
          launch_grid_iter(L, ctx->blocks.p + T.bk0, ctx->meta.p ? ctx->meta.p + static_cast<size_t>(T.bk0) * 32 : nullptr,
                           T.bk1 - T.bk0, T.gu0, T.gu1 - T.gu0, ctx->gstate.p, ctx->heavy.p, ctx->heavy_part.p,
                           ctx->heavy_cnt.p, ctx->params.p, ctx->pf.p, ctx->rank.p, sin, sout, ctx->unit_iters.p,
                           ctx->status.p, T.hot_begin, T.hot_rows, T.unit_rows, T.keep_stream,
                           sharded ? ctx->maxbuf.p : nullptr, s);
          LR_CUDA_TRY(cudaEventRecord(ctx->lev[static_cast<size_t>(k)], s));
          ++launches;
          ++spmv_launches;
          if (sharded) {
            // exchange step: every rank's s' shard to every rank (grouped
            // broadcasts = an in-place all-gather with uneven shards), and the
            // max of the shard maxima; then the same stop decision everywhere
            if (const lr_status xs = exchange_shards(ctx, T, sout, true); xs != LR_OK) return xs;
            launch_grid_finish(ctx->gstate.p, T.gu0, T.gu1 - T.gu0, ctx->params.p, ctx->unit_iters.p, ctx->status.p,
                               ctx->maxbuf.p, s);
            ++launches;
          }
        }
        LR_CUDA_TRY(cudaMemcpyAsync(ctx->h_status, ctx->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
        LR_CUDA_TRY(cudaStreamSynchronize(s));
        if (ctx->h_status->active <= 0 || k > cap + 2) break;
        // Next batch: the increments shrink geometrically, so the remaining
        // iterations follow from the last two maxima; enqueue them all (plus
        // one) so the level usually needs a single further poll.  Launches
        // past convergence exit at once.
        const double lm = ctx->h_status->last_max, pm = ctx->h_status->prev_max, tol = ctx->h_params->tol;
        int next = std::min(16, batch * 2);
        if (lm > 0.0 && pm > lm && lm >= tol) {
          const double rem = std::ceil(std::log(tol / lm) / std::log(lm / pm));
          if (rem >= 0.0 && rem < 4096.0) next = std::max(1, std::min(static_cast<int>(rem) + 1, 512));
        }
        batch = next;
      }
      LR_CUDA_TRY(cudaEventRecord(ctx->ev[3], s));
      LR_CUDA_TRY(cudaEventSynchronize(ctx->ev[3]));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
      spmv_ms += ms;
      if (ctx->unit_times) ctx->grid_level_ms[li] = ms;
      // roofline bookkeeping: per-unit iteration counts of this level
      const int ngu = T.gu1 - T.gu0;
      std::vector<GridUnitState> gsh(static_cast<size_t>(ngu));
      LR_CUDA_TRY(cudaMemcpy(gsh.data(), ctx->gstate.p + T.gu0, sizeof(GridUnitState) * ngu, cudaMemcpyDeviceToHost));
      long long kmax = 0;
      for (int i = 0; i < ngu; ++i) {
        const long long it = gsh[static_cast<size_t>(i)].iterations;
        kmax = std::max(kmax, it);
        spmv_bytes += it * (12 * ctx->gu_nnz[static_cast<size_t>(T.gu0 + i)] + 32 * ctx->gu_rows[static_cast<size_t>(T.gu0 + i)]);
        spmv_edges += it * ctx->gu_nnz[static_cast<size_t>(T.gu0 + i)];
      }
      if (std::min(kmax, k) > 0) {
        float lm = 0.f;
        cudaEventElapsedTime(&lm, ctx->lev[0], ctx->lev[static_cast<size_t>(std::min(kmax, k))]);
        active_ms += lm;
      }
      active_launches += std::min(kmax, k);
      // lower levels read these units' final ranks: replicate them on every rank
      if (ctx->comm)
        if (const lr_status xs = exchange_shards(ctx, T, ctx->rank.p, false); xs != LR_OK) return xs;
    }
  }
  launch_output(L, ctx->rank.p, r3_dev, ctx->partial.p, ctx->nparts, s);
  launch_normalize(r3_dev, r1_dev, ctx->n, ctx->partial.p, ctx->nparts, ctx->total.p, s);
  launches += 2 + (r1_dev ? 1 : 0);
  LR_CUDA_TRY(cudaGetLastError());
  LR_CUDA_TRY(cudaEventRecord(ctx->ev[1], s));
  if (prof_on) {
    LR_CUDA_TRY(set_level_prof(nullptr));
    static const char* names[5] = {"rows", "cac_warps", "cac_block", "small", "lcta"};
    std::fprintf(stderr, "[LR_LEVEL_PROF] k_level span sum %.1f us over %zu levels\n", prof_span, ctx->lt.size());
    if (side_levels)
      std::fprintf(stderr,
                   "[LR_LEVEL_PROF] %lld levels with a side stream: main %.1f us, side (row tasks + k_cac_big) %.1f us, "
                   "sum of per-level max %.1f us, side longer in %lld levels\n",
                   side_levels, side_main * 1e3, side_side * 1e3, side_crit * 1e3, side_longer);
    for (auto& e : pev) cudaEventDestroy(e);
    for (int ty = 0; ty < 5; ++ty)
      std::fprintf(stderr, "  %-10s ctas %8lld  sum of per-level max %9.1f us  critical in levels: %9.1f us\n",
                   names[ty], prof_cnt[ty], prof_max[ty], prof_crit[ty]);
  }
  if (ctx->dist_any) {
    // split units' iteration counts live on their owners (others hold 0; grid
    // units the same value everywhere), errors on whichever rank saw them
    const NcclApi& nc = nccl();
    LR_NCCL_TRY(nc.group_start());
    if (ctx->n_units > 0)
      LR_NCCL_TRY(nc.all_reduce(ctx->unit_iters.p, ctx->unit_iters.p, static_cast<size_t>(ctx->n_units), ncclInt64,
                                ncclMax, ctx->comm, s));
    LR_NCCL_TRY(nc.all_reduce(&ctx->status.p->err, &ctx->status.p->err, 1, ncclUint32, ncclMax, ctx->comm, s));
    LR_NCCL_TRY(nc.group_end());
  }
  LR_CUDA_TRY(cudaMemcpyAsync(ctx->h_status, ctx->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
  std::vector<int64_t> dist_iters;
  int64_t* iters_out = unit_iters;
  if (ctx->dist_any && ctx->n_units > 0 && !iters_out) {
    dist_iters.resize(static_cast<size_t>(ctx->n_units));
    iters_out = dist_iters.data();
  }
  if (iters_out && ctx->n_units > 0)
    LR_CUDA_TRY(cudaMemcpyAsync(iters_out, ctx->unit_iters.p, ctx->unit_iters.bytes(), cudaMemcpyDeviceToHost, s));
  LR_CUDA_TRY(cudaStreamSynchronize(s));
  if (ctx->dist_any) {  // the power-series totals from the reduced per-unit counts
    DevStatus& hs = *ctx->h_status;
    hs.total_iterations = 0;
    hs.iterative_edge_work = 0;
    for (int64_t u = 0; u < ctx->n_units; ++u)
      if (ctx->h_unit_kind[static_cast<size_t>(u)] == 3) {
        hs.total_iterations += iters_out[u];
        hs.iterative_edge_work += iters_out[u] * ctx->h_unit_edges[static_cast<size_t>(u)];
      }
  }
  float dev_ms = 0.f;
  cudaEventElapsedTime(&dev_ms, ctx->ev[0], ctx->ev[1]);
  if (ctx->unit_times) {  // per unit: span from its first task's start to its last task's end
    std::vector<long long> ht(ctx->ut_tasks.n), hc(ctx->ut_cacs.n);
    LR_CUDA_TRY(cudaMemcpy(ht.data(), ctx->ut_tasks.p, ctx->ut_tasks.bytes(), cudaMemcpyDeviceToHost));
    LR_CUDA_TRY(cudaMemcpy(hc.data(), ctx->ut_cacs.p, ctx->ut_cacs.bytes(), cudaMemcpyDeviceToHost));
    const size_t nu = static_cast<size_t>(ctx->n_units);
    std::vector<long long> lo(nu, 0), hi(nu, 0);
    auto add = [&](int32_t u, long long a, long long b) {
      if (a <= 0 || b < a) return;
      const size_t k = static_cast<size_t>(u);
      lo[k] = lo[k] ? std::min(lo[k], a) : a;
      hi[k] = std::max(hi[k], b);
    };
    for (size_t t = 0; t + 1 < ctx->task_unit_ptr.size(); ++t)
      for (int64_t j = ctx->task_unit_ptr[t]; j < ctx->task_unit_ptr[t + 1]; ++j)
        add(ctx->task_units[static_cast<size_t>(j)], ht[3 * t + 1], ht[3 * t + 2]);
    for (size_t i = 0; i < ctx->cac_unit.size(); ++i) add(ctx->cac_unit[i], hc[3 * i + 1], hc[3 * i + 2]);
    ctx->h_unit_ms.assign(nu, 0.0);
    for (size_t u = 0; u < nu; ++u) {
      if (hi[u] > lo[u]) ctx->h_unit_ms[u] = static_cast<double>(hi[u] - lo[u]) * 1e-6;
      if (ctx->h_unit_kind[u] == 3 && !ctx->grid_level_ms.empty())
        ctx->h_unit_ms[u] += ctx->grid_level_ms[static_cast<size_t>(ctx->level_of_unit[u])];
    }
    ctx->unit_ms_valid = true;
  }
  ctx->launches += launches;
  ctx->spmv_launches += spmv_launches;
  const DevStatus& st = *ctx->h_status;
  if (info) {
    info->total_iterations = st.total_iterations;
    info->iterative_edge_work = st.iterative_edge_work;
    info->all_weights_zero = st.wmax_bits == 0ull;
    info->n_devices = 1;
    info->device_ms = dev_ms;
    info->spmv_ms = spmv_ms;
    info->spmv_launches = spmv_launches;
    info->kernel_launches = launches;
    info->spmv_active_launches = active_launches;
    info->spmv_active_ms = active_ms;
    info->spmv_bytes = spmv_bytes;
    info->spmv_edges = spmv_edges;
  }
  if (st.err & kErrNegW) {
    lrerr::set("weights must be non-negative");
    return LR_EINVAL;
  }
  if (st.err & kErrNoConv) {
    lrerr::set("power series failed to converge");
    return LR_ENOCONV;
  }
  if (st.err & kErrDegen) {
    lrerr::set("dense solve degenerated numerically");
    return LR_EDEGEN;
  }
  return LR_OK;
}

lr_status lr_solve_device(lr_ctx* ctx, const double* w_dev, double c, double tol, double* r3_dev, double* r1_dev,
                          lr_solve_info* info, int64_t* unit_iters) {
  return solve_on_device(ctx, w_dev, c, tol, r3_dev, r1_dev, info, unit_iters);
}

lr_status lr_solve(lr_ctx* ctx, const double* w, double c, double tol, double* r3, double* r1, lr_solve_info* info,
                   int64_t* unit_iters) {
  if (!ctx || !ctx->loaded) {
    lrerr::set("context has no uploaded layout");
    return LR_EINVAL;
  }
  LR_CUDA_TRY(cudaSetDevice(ctx->device));
  const size_t bytes = static_cast<size_t>(ctx->n) * sizeof(double);
  if (bytes) LR_CUDA_TRY(h2d_async(ctx->w.p, w, bytes, ctx->stream));
  if (std::getenv("LR_PROBE_SYNC")) LR_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  const lr_status st = solve_on_device(ctx, ctx->w.p, c, tol, ctx->r3.p, ctx->r1.p, info, unit_iters);
  if (st != LR_OK && st != LR_ENOCONV && st != LR_EDEGEN) return st;
  if (bytes) {
    if (host_pinned(r3) && (!r1 || host_pinned(r1))) {
      LR_CUDA_TRY(cudaMemcpyAsync(r3, ctx->r3.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
      if (r1) LR_CUDA_TRY(cudaMemcpyAsync(r1, ctx->r1.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
      LR_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    } else {
      LR_CUDA_TRY(d2h_sync(r3, ctx->r3.p, bytes, ctx->stream));
      if (r1) LR_CUDA_TRY(d2h_sync(r1, ctx->r1.p, bytes, ctx->stream));
    }
  }
  return st;
}

lr_status lr_nccl_unique_id(char* out128) {
  const NcclApi& nc = nccl();
  if (!nc.ok) {
    lrerr::set("libnccl.so.2 not loadable");
    return LR_ENCCL;
  }
  ncclUniqueId id;
  LR_NCCL_TRY(nc.get_unique_id(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof id);
  return LR_OK;
}

lr_status lr_ctx_set_comm(lr_ctx* ctx, int rank, int world, const char* id128) {
  if (!ctx || world < 1 || rank < 0 || rank >= world) {
    lrerr::set("bad rank / world");
    return LR_EINVAL;
  }
  if (world > 1 && !id128) {
    lrerr::set("world > 1 needs the NCCL unique id of rank 0");
    return LR_EINVAL;
  }
  ncclComm_t comm = nullptr;
  if (world > 1 || id128) {
    const NcclApi& nc = nccl();
    if (!nc.ok) {
      lrerr::set("libnccl.so.2 not loadable");
      return LR_ENCCL;
    }
    LR_CUDA_TRY(cudaSetDevice(ctx->device));
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    LR_NCCL_TRY(nc.comm_init_rank(&comm, world, id, rank));
  }
  // commit only once the new communicator exists
  if (ctx->comm) nccl().comm_destroy(ctx->comm);
  ctx->comm = comm;
  ctx->shard = rank;
  ctx->nshards = world;
  ctx->loaded = false;  // the next upload shards the grid units
  return LR_OK;
}

lr_status lr_ctx_unit_times(const lr_ctx* ctx, double* ms, int64_t n) {
  if (!ctx || !ms || !ctx->unit_ms_valid || n != ctx->n_units) {
    lrerr::set("no per-unit times: upload with LR_UNIT_TIMES=1, then solve");
    return LR_EINVAL;
  }
  std::copy(ctx->h_unit_ms.begin(), ctx->h_unit_ms.end(), ms);
  return LR_OK;
}

lr_status lr_split_level_rows(const int64_t* iptr, const int64_t* xptr, const int32_t* unit_row_begin,
                              const uint8_t* unit_kind, int32_t unit_begin, int32_t unit_end, int32_t world,
                              int32_t* bounds) {
  if (!iptr || !xptr || !unit_row_begin || !unit_kind || !bounds || world < 1 || unit_end < unit_begin) {
    lrerr::set("bad level split request");
    return LR_EINVAL;
  }
  const std::vector<int> b = split_level_rows(iptr, xptr, unit_row_begin, unit_kind, unit_begin, unit_end, world);
  std::copy(b.begin(), b.end(), bounds);
  return LR_OK;
}

lr_status lr_exchange_cuts(const int64_t* iptr, int32_t row_begin, int32_t row_end, int32_t world, int32_t chunks,
                           int32_t* cuts) {
  if (!iptr || !cuts || world < 1 || chunks < 1 || row_end < row_begin) {
    lrerr::set("bad exchange request");
    return LR_EINVAL;
  }
  const std::vector<int> c = exchange_cuts(iptr, row_begin, row_end, world, chunks);
  std::copy(c.begin(), c.end(), cuts);
  return LR_OK;
}

lr_status lr_shard_rows(const int64_t* iptr, int32_t row_begin, int32_t row_end, int32_t world, int32_t* bounds) {
  if (!iptr || !bounds || world < 1 || row_end < row_begin) {
    lrerr::set("bad shard request");
    return LR_EINVAL;
  }
  const std::vector<int> b = shard_bounds(iptr, row_begin, row_end, world);
  std::copy(b.begin(), b.end(), bounds);
  return LR_OK;
}

lr_status lr_propagate_weights(int device, const int32_t* src, const int32_t* dst, const int32_t* deg, int64_t m,
                               const double* ranks, int64_t n, double c, double* weights) {
  for (int64_t i = 0; i < m; ++i)
    if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n || deg[i] <= 0) {
      lrerr::set("cross edge out of range");
      return LR_EINVAL;
    }
  // stable grouping by destination (input order kept within a destination)
  std::vector<long long> cnt(static_cast<size_t>(n) + 1, 0);
  for (int64_t i = 0; i < m; ++i) ++cnt[static_cast<size_t>(dst[i]) + 1];
  for (int64_t v = 0; v < n; ++v) cnt[static_cast<size_t>(v) + 1] += cnt[static_cast<size_t>(v)];
  std::vector<int> order(static_cast<size_t>(m));
  {
    std::vector<long long> cur(cnt.begin(), cnt.end() - 1);
    for (int64_t i = 0; i < m; ++i) order[static_cast<size_t>(cur[static_cast<size_t>(dst[i])]++)] = static_cast<int>(i);
  }
  std::vector<long long> seg;
  for (int64_t v = 0; v < n; ++v)
    if (cnt[static_cast<size_t>(v) + 1] > cnt[static_cast<size_t>(v)]) seg.push_back(cnt[static_cast<size_t>(v)]);
  seg.push_back(m);
  lr_ctx* ctx = nullptr;
  lr_status st = lr_ctx_create(device, &ctx);
  if (st != LR_OK) return st;
  cudaStream_t s = ctx->stream;
  DevBuf<int> d_src, d_dst, d_deg, d_order;
  DevBuf<long long> d_seg;
  DevBuf<double> d_r, d_w;
  auto run = [&]() -> lr_status {
    LR_CUDA_TRY(d_src.upload(src, static_cast<size_t>(m), s));
    LR_CUDA_TRY(d_dst.upload(dst, static_cast<size_t>(m), s));
    LR_CUDA_TRY(d_deg.upload(deg, static_cast<size_t>(m), s));
    LR_CUDA_TRY(d_order.upload(order.data(), order.size(), s));
    LR_CUDA_TRY(d_seg.upload(seg.data(), seg.size(), s));
    LR_CUDA_TRY(d_r.upload(ranks, static_cast<size_t>(n), s));
    LR_CUDA_TRY(d_w.upload(weights, static_cast<size_t>(n), s));
    launch_propagate(d_order.p, d_seg.p, static_cast<int>(seg.size()) - 1, d_src.p, d_dst.p, d_deg.p, d_r.p, c, d_w.p, s);
    LR_CUDA_TRY(cudaGetLastError());
    if (n) LR_CUDA_TRY(cudaMemcpyAsync(weights, d_w.p, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost, s));
    LR_CUDA_TRY(cudaStreamSynchronize(s));
    return LR_OK;
  };
  st = run();
  d_src.reset();
  d_dst.reset();
  d_deg.reset();
  d_order.reset();
  d_seg.reset();
  d_r.reset();
  d_w.reset();
  lr_ctx_free(ctx);
  return st;
}

}  // extern "C"
