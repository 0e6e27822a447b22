// Device kernels of the level-scheduled PageRank solve (sm_100a).  See
// DESIGN.md "Kernels" for each kernel's roofline and algorithmic bytes.
#pragma once

#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <vector>

namespace lrk {

// per-row kind (uploaded once)
enum RowKind : std::uint8_t { kSingle = 0, kCac = 1, kSmall = 2, kLargeCta = 3, kLargeGrid = 4 };

// device-side error bits
enum ErrBits : unsigned { kErrNoConv = 1u, kErrDegen = 2u, kErrNegW = 4u, kErrCycle = 8u };

// Per-solve scalars, read by every kernel from global memory.
struct SolveParams {
  double c;
  double tol;
  long long cap;  // iteration_cap (solvers.cpp:17-21)
};

// Small device-side status block (one per context).
struct DevStatus {
  unsigned err;
  int all_zero;            // max(w) == 0
  unsigned long long wmax_bits;
  long long total_iterations;
  long long iterative_edge_work;
  int active;              // grid SccLarge units still iterating on the current level
  int ctas_done;           // CTAs finished with the running grid SpMV launch
  double last_max;         // largest max|inc| over the level's running units, latest closed iteration
  double prev_max;         // the same one iteration earlier (host predicts the remaining iterations)
  int next_task;           // k_spmv_seg: next unclaimed task of the running launch (reset by its last CTA)
  int pad;
};

// One SccLarge grid unit's iteration state.
struct GridUnitState {
  unsigned long long max_bits;  // max(y) of the running iteration (y >= 0)
  int iterations;
  int done;
  int unit;                     // schedule unit index (for unit_iters)
  int nblocks;
  long long edges;              // reference unit.edges.size()
};

// A row block of the grid SpMV: rows [row_begin, row_end) of one unit, or one
// segment of a heavy row (heavy >= 0).
struct SpmvBlock {
  long long nnz_begin;  // first in-edge of the block (absolute, into isrc)
  int nnz;              // in-edges in the block (<= kSpmvNnz)
  int row_begin;
  int row_end;
  int gunit;            // index into GridUnitState array
  int heavy;            // heavy-row id or -1
  int seg;              // segment index within the heavy row
};

struct HeavyRow {
  int row;
  int nseg;
  long long part_begin;  // into heavy partial buffer
};

struct DeviceLayout {
  int n;
  const int* vertex_of;
  const int* row_of;
  const int* deg;
  const std::uint8_t* loop;
  const std::uint8_t* rowkind;
  const long long* xptr;
  const int* xsrc;
  const long long* iptr;
  const int* isrc;
};

// tasks: CAC unit = rows [row_begin,row_end) with depth slices
struct CacTask {
  int row_begin;
  int row_end;
  long long depth_begin;  // into depth_ptr
  int ndepth;
  int pregathered;  // start weights gathered by row tasks launched before (k_cac_big skips its own)
};
struct SccTask {
  int row_begin;
  int row_end;
  int unit;
  int pad;
  long long edges;
};

// A slice of one heavy row's cross in-edges (rows with more than kCrossLight).
struct CrossTask {
  long long e_begin;     // into xsrc
  long long part_begin;  // partial slots of the row (nseg > 1)
  int cnt;
  int row;
  int seg;
  int nseg;
  int slot;              // completion counter of the row
  int pad;
};

constexpr int kCrossLight = 32;    // rows up to this many in-edges: one thread, reference order
constexpr int kCrossSplit = 32;    // cross rows above this: split over warps by k_pull_heavy
constexpr int kCrossSeg = 256;     // in-edges per warp task of a split row (8 per lane, all in flight)
constexpr int kTileNnzCross = 256; // cross in-edges per chunk of a row task (level.cu cross_rows_tiled)
constexpr size_t kRowTaskSmem = 8 * kTileNnzCross * sizeof(double);  // k_level smem a row task needs
constexpr size_t kBigCrossSmem = 32 * kTileNnzCross * sizeof(double);  // k_cac_big's warp-tiled start weights
constexpr int kCacPregatherRows = 1024;  // larger CACs (all of k_cac_big's): start weights by row tasks first
                                         // (config 4: 34.6 ms at 4096, 32.1 ms at 2048 and 1024)

// One CTA of the fused per-level kernel (level.cu).
enum LevelTaskType : int {
  kTaskRows = 0,
  kTaskCacWarps = 1,
  kTaskCacBlock = 2,
  kTaskSmall = 3,
  kTaskLcta = 4,
  // start weights split across two levels (config-4 shaped chains): the terms
  // from sources in rows below `split` (levels solved at least two levels
  // earlier, a prefix of every row's ordered cross list) summed one level
  // early into xpart; the rest added from xpart at the row's own level
  kTaskRowsPart = 5,
  kTaskRowsFin = 6,
};
constexpr int kTaskTypes = 7;
struct LevelTask {
  int type;
  int a;      // rows: first row; CAC warps: first CacTask; others: task index
  int b;      // rows: end row; CAC warps: end CacTask
  int split;  // kTaskRowsPart / kTaskRowsFin: first row of the level solved just before the rows' own
};
constexpr int kCacBlockMaxRows = 32768;  // larger CACs: one grid-wide launch per depth slice
#ifndef LR_SPMV_THREADS
#define LR_SPMV_THREADS 1024
#endif
constexpr int kSpmvThreads = LR_SPMV_THREADS;  // K4b: one persistent CTA per SM: 32 warps + a shared-memory head
#ifndef LR_SEG_THREADS
#define LR_SEG_THREADS 768
#endif
constexpr int kSegThreads = LR_SEG_THREADS;    // K4c: 24 warps per SM (78 registers, no spills)
constexpr int kTileNnz = 256;      // in-edges of one warp tile
constexpr int kTileRows = 64;      // max rows of one warp tile
constexpr int kSegNnz = 1024;      // rows above this are split into segments
// k_spmv_seg (spmv.cu): a chunk of <= kChunkNnz in-edges always lies inside the
// 32-byte aligned 256-slot window that starts at or below it, so one 256-bit
// index load per lane covers it; heavy-row segments are four chunks.
constexpr int kChunkNnz = 248;
constexpr int kChunkSegNnz = 4 * kChunkNnz;
constexpr int kIdxPad = 256;       // isrc is allocated this many entries past its end
constexpr int kMaxSharedUnits = 256;  // grid units whose done flags k_spmv_seg keeps in shared memory
constexpr int kCtaLargeMaxRows = 4096;
constexpr long long kCtaLargeMaxNnz = 1 << 16;
constexpr int kMaxDynSmem = 227 * 1024;
constexpr int kSmallSmemMaxM = 160;      // ld*(ld+2)*8 <= 227 KB
constexpr int kSmallScratchBlocks = 296; // grid of the global-scratch small-SCC path
constexpr int kSmallTileMaxM = 128;     // small SCCs up to this: tile Gauss-Jordan (level.cu)
// the fraction-free tile solve keeps minors of size down to (1-c)^m: use it
// while that stays far from underflow, else the normalised solve (level.cu)
__host__ __device__ inline bool small_tile_ok(int m, double c) {
  return m <= kSmallTileMaxM && static_cast<double>(m) * log1p(-c) > -640.0;
}
// shared memory of the tile solve: m x small_tile_ld(m) matrix, m solution values,
// the unit's ne in-edges (value + column)
__host__ __device__ constexpr int small_tile_ld(int m) { return (m + 32) | 1; }
// SccSmall units up to this many rows: block Gauss-Jordan on FP64 tensor cores
// (level.cu small_solve_mma); its shared memory: the 64 x 72 system, 64
// solution values, the unit's in-edges
constexpr int kSmallMmaMaxM = 64;
__host__ __device__ constexpr size_t small_mma_bytes(long long ne) {
  return (64 * 72 + 64) * sizeof(double) + static_cast<size_t>(ne) * (sizeof(double) + sizeof(int));
}
// up to this many rows: the block Gauss-Jordan with the system in shared memory
// (small_solve_mma_smem): mp x (mp + 8) system, mp x 8 column block, 8 x (mp + 8)
// row block, mp solution values, the in-edges (mp = m rounded up to 8)
constexpr int kSmallMmaSmemMaxM = 128;
__host__ __device__ constexpr size_t small_mma_smem_bytes(int m, long long ne) {
  return (static_cast<size_t>((m + 7) & ~7) * static_cast<size_t>(((m + 7) & ~7) + 16) +
          static_cast<size_t>((m + 7) & ~7) * 8 + 8 * static_cast<size_t>(((m + 7) & ~7) + 16) +
          static_cast<size_t>((m + 7) & ~7)) * sizeof(double) +
         static_cast<size_t>(ne) * (sizeof(double) + sizeof(int));
}
// shared memory of the small-SCC solve k_level picks for a unit
// (level.cu small_dispatch): block GJ in registers (m <= 64), block GJ with the
// system in shared memory (m <= 128), else the normalised GJ (no edge stash)
__host__ __device__ constexpr size_t small_unit_smem_bytes(int m, long long ne);
// k_level's dynamic shared memory ceiling (227 KB opt-in less its static
// shared memory, with margin); units above it run in the global-scratch k_small
constexpr size_t kSmallSmemCap = 232448 - 1024;
__host__ __device__ constexpr size_t small_tile_bytes(int m, long long ne) {
  return (static_cast<size_t>(m) * static_cast<size_t>(small_tile_ld(m)) + static_cast<size_t>(m)) * sizeof(double) +
         static_cast<size_t>(ne) * (sizeof(double) + sizeof(int));
}
__host__ __device__ constexpr size_t small_unit_smem_bytes(int m, long long ne) {
  return m <= kSmallMmaMaxM        ? small_mma_bytes(ne)
         : m <= kSmallMmaSmemMaxM ? small_mma_smem_bytes(m, ne)
                                   : static_cast<size_t>(m + 1) * static_cast<size_t>(m + 2) * sizeof(double);
}
// shared memory of lcta_solve_staged for a unit of m rows and ne in-edges,
// with the level's largest unit at maxrows rows
__host__ __device__ constexpr size_t lcta_stage_bytes(int maxrows, long long ne) {
  return static_cast<size_t>(maxrows) * 32 + ((static_cast<size_t>(maxrows) + 1) * 4 + 7) / 8 * 8 +
         static_cast<size_t>(ne) * 2;
}
constexpr size_t kLctaStageMaxBytes = 96 * 1024;  // k_level smem budget for staged CTA power series
#ifndef LR_LCTA_REGIDX
#define LR_LCTA_REGIDX 12
#endif
constexpr int kLctaRegIdx = LR_LCTA_REGIDX;  // in-edge offsets per row kept in registers by the CTA power series
constexpr int kLctaRegRows = 512;            // units up to this many rows: register rows (two per thread)
constexpr int kCacWarpMaxRows = 64;      // CACs up to this: one warp of a k_level CTA
constexpr int kCacMidMaxRows = 1024;     // up to this: a 256-thread k_level CTA; above: a 1024-thread CTA

cudaError_t configure_kernels();
cudaError_t configure_level_kernel();

// large CACs, 1024-thread CTAs, meant for a second stream (level.cu)
void launch_cac_big(const DeviceLayout& L, const CacTask* cacs, int n, const int* depth_ptr, const double* w,
                    const SolveParams* p, const double* pf, double* rank, double* s0, double* pv, size_t smem,
                    cudaStream_t s, long long* task_times = nullptr);
// shared-memory bytes a CAC of `rows` rows and `edges` in-edges needs to be swept from shared memory
size_t cac_stage_need(long long rows, long long edges);
size_t cac_compact_need(long long rows, long long edges);  // k_cac_big's structure-only staging
constexpr size_t kStageMaxBytes = 200 * 1024;  // larger CACs sweep from global memory
constexpr size_t kLevelStageBytes = 64 * 1024; // CAC staging budget of one k_level CTA
// k_level per-CTA timing buffer (3 int64 per CTA: type, start ns, end ns), nullptr = off
cudaError_t set_level_prof(long long* buf);
// fused per-level kernel (level.cu)
void launch_level(const DeviceLayout& L, const LevelTask* tasks, int ntasks, const CacTask* cacs, const int* depth_ptr,
                  const SccTask* smalls, const SccTask* lctas, int small_ld, int lcta_rows, size_t smem,
                  const double* w, const SolveParams* p, const double* pf, double* rank, double* s0,
                  long long* unit_iters, DevStatus* st, bool heavy, cudaStream_t s, bool profile = true,
                  double* xpart = nullptr, long long* task_times = nullptr);

// launch wrappers (stream-ordered)
void launch_prep(const DeviceLayout& L, const double* w, const SolveParams* p, double* pf, DevStatus* st,
                 cudaStream_t s);
void launch_cross_heavy(const DeviceLayout& L, const CrossTask* tasks, int ntasks, const double* w,
                        const SolveParams* p, const double* pf, double* rank, double* s0, double* parts, int* cnts,
                        cudaStream_t s);
void launch_cac_slice(const DeviceLayout& L, int row_begin, int row_end, const SolveParams* p, double* rank,
                      cudaStream_t s);
void launch_cac_heavy(const DeviceLayout& L, const CrossTask* tasks, int ntasks, const SolveParams* p, double* rank,
                      double* parts, int* cnts, cudaStream_t s);
void launch_small(const DeviceLayout& L, const SccTask* tasks, int ntasks, int max_m, const double* pf,
                  double* rank, double* scratch, DevStatus* st, cudaStream_t s);
void launch_grid_reset(GridUnitState* gs, int ngu, DevStatus* st, cudaStream_t s);
int grid_iter_ctas();
bool spmv_seg();  // K4c segmented-scan SpMV (default) or K4b staged tiles (LR_SPMV=tile)
// meta: per task 32 lane words (row-start flags of the lane's 8 slots | rows
// starting before them << 8) for k_spmv_seg tiles (build_chunk_meta)
void launch_grid_iter(const DeviceLayout& L, const SpmvBlock* blocks, const unsigned short* meta, int nblocks, int gu0,
                      int ngu, GridUnitState* gs,
                      const HeavyRow* heavy, double* heavy_part, int* heavy_cnt, const SolveParams* p,
                      const double* pf, double* rank, const double* s_in, double* s_out, long long* unit_iters,
                      DevStatus* st, int hot_begin, long long hot_rows, long long unit_rows, int keep_stream,
                      double* maxbuf, cudaStream_t s, int hold = 0);
// multi-GPU: close an iteration from the all-reduced shard maxima in maxbuf
void launch_grid_finish(GridUnitState* gs, int gu0, int ngu, const SolveParams* p, long long* unit_iters,
                        DevStatus* st, const double* maxbuf, cudaStream_t s);
void launch_grid_zero_max(double* maxbuf, int gu0, int ngu, cudaStream_t s);
void launch_output(const DeviceLayout& L, const double* rank, double* r3, double* partial, int nparts,
                   cudaStream_t s);
void launch_normalize(const double* r3, double* r1, int n, const double* partial, int nparts, double* total,
                      cudaStream_t s);
void launch_propagate(const int* dst_order, const long long* seg_ptr, int nseg, const int* src, const int* dst,
                      const int* deg, const double* ranks, double c, double* weights, cudaStream_t s);

// K5 (k_spmv_blk, spmv.cu): the power-series SpMV of one large grid unit in
// dest-row blocks.  Block b = unit rows [b*BR, (b+1)*BR); its in-edges sorted by
// source (esrc: source row in the unit, edst: dest row in the block) in slots of
// kBlkChunk; unused slots hold (src 0, dst BR) dummies, which K5 skips.  Inside
// a window of kBlkWindow slots the entries are placed so that each half-warp's
// dest rows fall on distinct shared-memory bank pairs (blk.cu).  A part is a
// contiguous range of one block's slots; blocks with several parts add their
// partial rows into yacc (slot) and the last part to finish closes the rows.
#ifndef LR_BLK_THREADS
#define LR_BLK_THREADS 1024
#endif
constexpr int kBlkThreads = LR_BLK_THREADS;
constexpr int kBlkChunk = 256;    // slots per warp step (8 per lane, lane-strided)
constexpr int kBlkWindow = 8192;  // slots the bank balance looks at together (blk.cu k_blk_banks)
constexpr int kBlkSlack = 32;     // rows of 32 entries per empty row (0: none)
constexpr int kBlkReach = 1 << 20;  // rows a left-over entry looks at on either side for a conflict-free slot
struct BlkPart {
  long long e0;  // first entry (into esrc/edst)
  int n;         // entries (multiple of kBlkChunk)
  int blk;       // dest block
  int slot;      // split blocks: partial-row slot, else -1
  int nsplit;    // parts of the block
};
struct BlkUnitDev {
  const unsigned* esrc;
  const unsigned short* edst;
  const BlkPart* parts;
  int nparts;
  int u0;    // first row of the unit (sources are unit-relative)
  int UR;    // rows of the unit
  int row0;  // first dest row of this layout (u0, or a shard chunk's first row)
  int R;     // dest rows of this layout
  int BR;    // rows per block
  double* yacc;  // [split blocks][BR]
  int* bcnt;     // [split blocks]
};
// entries of rows [u0, u0 + R) (CSR iptr/isrc on the device, in-edges
// [e_begin, e_begin + E)) sorted by (block, source): block b's run lands at
// pad_off[b] (host array, NB + 1 entries, multiples of kBlkChunk), one empty row
// of 32 slots after every `slack` rows, bank-balanced in windows of `win` slots
// (row0, R: the dest rows; u0, UR: the unit, whose rows the sources index)
cudaError_t build_blk_entries(const long long* iptr, const int* isrc, long long e_begin, long long E, int u0, int UR,
                              int row0, int R, int BR, const std::vector<long long>& pad_off, int slack, int win,
                              unsigned* esrc, unsigned short* edst, cudaStream_t s);
// maxbuf / hold: the row-sharded protocol of launch_grid_iter
void launch_spmv_blk(const BlkUnitDev& B, int gu, GridUnitState* gs, const SolveParams* p, const double* pf,
                     double* rank, const double* s_in, double* s_out, long long* unit_iters, DevStatus* st,
                     int hot_begin, long long hot_rows, long long unit_rows, cudaStream_t s, double* maxbuf = nullptr,
                     int hold = 0);

constexpr int kOutBlock = 1024;  // rows per partial sum of the R1 normalisation

}  // namespace lrk
