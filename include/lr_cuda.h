/* levelrank-b200: the C-ABI drop-in boundary of the level-scheduled PageRank
 * solve (arXiv 1609.09068).  Plain pointers and sizes only; no C++ or torch
 * types; no exception crosses it.  Every entry point names the reference
 * interface (/root/reference/proj/...) it replaces.  The C++ host API in
 * include/levelrank/ headers and the Python package paper_1609_09068_b200 are both
 * thin layers over these symbols; INTEGRATION.md shows the bindings.
 *
 * Status codes map back to the reference's exceptions:
 *   LR_EINVAL  -> std::invalid_argument   (solvers.cpp:11-15, engine.cpp:94-97, schedule.cpp:33)
 *   LR_ENOCONV -> std::runtime_error("power series failed to converge")  (solvers.cpp:159)
 *   LR_ECYCLE  -> std::logic_error("cycle inside an acyclic component")  (solvers.cpp:84-85)
 *   LR_EDEGEN  -> std::runtime_error("dense solve degenerated numerically") (solvers.cpp:103-106)
 *   LR_EIO     -> IoError / ParseError (graph.hpp:26-35)
 *   LR_ECUDA / LR_ENCCL / LR_ENOMEM -> std::runtime_error(lr_last_error())
 * lr_last_error() returns a thread-local message for the last failure.
 */
#ifndef LR_CUDA_H
#define LR_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum lr_status {
  LR_OK = 0,
  LR_EINVAL = 1,
  LR_ENOCONV = 2,
  LR_ECYCLE = 3,
  LR_EDEGEN = 4,
  LR_ECUDA = 5,
  LR_ENCCL = 6,
  LR_ENOMEM = 7,
  LR_EIO = 8
} lr_status;

const char* lr_last_error(void);
const char* lr_version(void);

/* ------------------------------------------------------------ graph core */
typedef struct lr_graph lr_graph;

/* Graph::from_edges (proj/src/graph.cpp:14-36): range check, dedup, sorted
 * rows, loop flags.  keep_loops selects LoopPolicy::Keep (graph.hpp:23). */
lr_status lr_graph_from_edges(int32_t n, const int32_t* src, const int32_t* dst, int64_t m,
                              int keep_loops, lr_graph** out);
/* Adopt a CSR with sorted, duplicate-free rows (checked). */
lr_status lr_graph_from_csr(int32_t n, const int64_t* offsets, const int32_t* targets,
                            int keep_loops, lr_graph** out);
/* load_edge_list (proj/src/graph.cpp:101-105 -> parse_edge_list :54-99):
 * the file is mmap'ed and parsed by all host threads; LR_EIO with
 * "line N: ..." for the first malformed line, as the reference reports it. */
lr_status lr_graph_load_edge_list(const char* path, int dense_ids, int keep_loops, lr_graph** out);
/* parse_edge_list (proj/src/graph.cpp:54-99) over an in-memory byte buffer. */
lr_status lr_graph_parse_edge_buffer(const char* data, int64_t len, int dense_ids, int keep_loops,
                                     lr_graph** out);
int32_t lr_graph_vertex_count(const lr_graph* g);
int64_t lr_graph_edge_count(const lr_graph* g);
/* CSR export; any pointer may be NULL.  walk_deg = Graph::walk_out_degree. */
lr_status lr_graph_csr(const lr_graph* g, int64_t* offsets, int32_t* targets, uint8_t* has_loop,
                       int32_t* walk_deg);
void lr_graph_free(lr_graph* g);

/* ------------------------------------------------------------- partition */
/* find_components / find_components_scc_only (proj/src/partition.cpp:246-250).
 * comp_of[n]; kinds/levels/sizes need capacity n (k entries written);
 * kinds: 0 = Scc, 1 = Cac.  stats3 (nullable): explore_edge_visits,
 * merge_scan_edge_visits, finish_calls (partition.hpp:31-35). */
lr_status lr_find_components(const lr_graph* g, int merge_cacs, int32_t* comp_of, int32_t* kinds,
                             int32_t* levels, int32_t* sizes, int32_t* k_out, int32_t* max_level,
                             int64_t* stats3);

/* ------------------------------------------------------------------ plan */
/* A plan = find_components + build_schedule + the device Layout, built on the
 * host (multi-threaded).  Replaces the two calls at proj/src/engine.cpp:114-115.
 * The plan borrows g; g must outlive it. */
typedef struct lr_plan lr_plan;
lr_status lr_plan_build(const lr_graph* g, int32_t small_threshold, lr_plan** out);
/* The whole graph as one power-series unit: the layout of compute_baseline
 * (proj/src/engine.cpp:184-218, solve_baseline proj/src/solvers.cpp:164-198),
 * no partition and no schedule (those views return LR_EINVAL).  Upload and
 * solve it like any plan; the unit's iteration count is the baseline's. */
lr_status lr_plan_build_baseline(const lr_graph* g, lr_plan** out);
void lr_plan_free(lr_plan* p);

/* The reference Schedule (proj/include/levelrank/schedule.hpp:13-57), flattened
 * level-major for parity checks.  out8 = [n_levels, n_units, n_ids, n_edges,
 * n_cross, intra_edge_count, cross_edge_count, dropped_loop_count]. */
lr_status lr_plan_schedule_sizes(const lr_plan* p, int64_t* out8);
lr_status lr_plan_schedule_get(const lr_plan* p, int32_t* level_values, int32_t* level_unit_begin,
                               int64_t* level_cross_begin, int32_t* unit_kind, int32_t* unit_level,
                               int32_t* unit_size, int64_t* unit_ids_begin,
                               int64_t* unit_edges_begin, int32_t* ids, int32_t* edge_src,
                               int32_t* edge_dst, int32_t* cross_src, int32_t* cross_dst,
                               int32_t* cross_deg, int32_t* permutation);

/* PartitionCensus (partition.hpp:65-78) of the plan's partition. */
typedef struct lr_census {
  int64_t components, scc_components, cac_components, singleton_cacs;
  int32_t largest_component, largest_is_scc, max_level, level_count;
} lr_census;
lr_status lr_plan_census(const lr_plan* p, lr_census* out);

/* Borrowed view of the device Layout (levelrank::Layout, schedule.hpp).  All
 * arrays are in row (level-major) order; see DESIGN.md "Data layout in HBM". */
typedef struct lr_layout {
  int32_t n;
  int32_t n_levels;
  int32_t keep_loops;
  int64_t n_units;
  int64_t nnz_cross;
  int64_t nnz_intra;
  int64_t depth_ptr_len;
  const int32_t* level_row_begin;  /* n_levels + 1 */
  const int32_t* level_unit_begin; /* n_levels + 1 */
  const int32_t* vertex_of;        /* n */
  const int32_t* row_of;           /* n */
  const int32_t* deg;              /* n, walk out-degree */
  const uint8_t* loop;             /* n */
  const int64_t* xptr;             /* n + 1 */
  const int32_t* xsrc;             /* nnz_cross */
  const int64_t* iptr;             /* n + 1 */
  const int32_t* isrc;             /* nnz_intra */
  const uint8_t* unit_kind;        /* n_units: 0 Singleton, 1 Cac, 2 SccSmall, 3 SccLarge */
  const int32_t* unit_level;       /* n_units */
  const int32_t* unit_row_begin;   /* n_units + 1 */
  const int64_t* unit_edges;       /* n_units */
  const int64_t* cac_depth_begin;  /* n_units */
  const int32_t* depth_ptr;        /* depth_ptr_len */
} lr_layout;
lr_status lr_plan_layout(const lr_plan* p, lr_layout* out);

/* --------------------------------------------------------- device solve */
typedef struct lr_ctx lr_ctx;

/* Per-solve figures reported beside SolveReport. */
typedef struct lr_solve_info {
  int64_t total_iterations;   /* sum of SccLarge iterations (engine.cpp:160-163) */
  int64_t iterative_edge_work;/* sum over SccLarge units of iterations * unit edges */
  int32_t all_weights_zero;   /* engine.cpp:112 */
  int32_t n_devices;
  double device_ms;           /* CUDA-event time of the whole device solve */
  double spmv_ms;             /* CUDA-event time inside grid-wide SccLarge iterations */
  int64_t spmv_launches;      /* grid-wide SccLarge iteration launches */
  int64_t kernel_launches;    /* all kernels this solve launched */
  /* roofline evidence for the dominant kernel (grid SpMV), from per-launch
   * CUDA events: launches that still had a running unit, their summed device
   * time, and the algorithmic bytes they moved (12 B per in-edge + 32 B per
   * row of every unit still iterating). */
  int64_t spmv_active_launches;
  double spmv_active_ms;
  int64_t spmv_bytes;
  int64_t spmv_edges;         /* edge updates done by those launches */
} lr_solve_info;

/* One context per host thread; owns device memory and a stream on `device`. */
lr_status lr_ctx_create(int device, lr_ctx** out);
/* Uploads a layout; replaces any previous one.  Builds the per-kernel task
 * tables (SccLarge row blocks, CAC / small-SCC task lists). */
lr_status lr_ctx_upload(lr_ctx* ctx, const lr_layout* layout);
/* The level loop of compute_pagerank (proj/src/engine.cpp:126-158) on the GPU,
 * then R1 = R3 / ||R3||_1 (the normalisation of oracle_r1_to_r3,
 * solvers.cpp:200-244).  Host buffers in vertex-id order: w (n), r3 (n),
 * r1 (n, nullable).  unit_iters (nullable, n_units) receives per-unit
 * iteration counts in schedule order (0 for one-pass kinds).  Validates
 * params and weights like engine.cpp:92-97. */
lr_status lr_solve(lr_ctx* ctx, const double* w, double c, double tol, double* r3, double* r1,
                   lr_solve_info* info, int64_t* unit_iters);
/* Same with device-resident buffers (vertex-id order, on ctx's device);
 * unit_iters stays a host pointer.  Stream-ordered on lr_ctx_stream(). */
lr_status lr_solve_device(lr_ctx* ctx, const double* w_dev, double c, double tol, double* r3_dev,
                          double* r1_dev, lr_solve_info* info, int64_t* unit_iters);
/* ------------------------------------------------------------ multi-GPU */
/* The grid-wide SccLarge units (the giant SCC) can be row-sharded over the
 * GPUs of one node (the reference is single-process,
 * SPEC.md:383).  Every rank builds the same plan and calls lr_ctx_set_comm
 * before lr_ctx_upload; each rank then iterates only its nnz-balanced row
 * shard, and after every iteration the shards of s' are exchanged in place
 * over NCCL (grouped broadcasts) together with an all-reduce(max) of the shard
 * maxima, so every rank takes the same stop decision.  All other units are
 * solved redundantly on every rank; results are identical on all ranks. */
lr_status lr_nccl_unique_id(char* out128);
lr_status lr_ctx_set_comm(lr_ctx* ctx, int rank, int world, const char* unique_id128);
/* The nnz-balanced split used for the shards: bounds[world + 1] over rows
 * [row_begin, row_end) of a pull CSR with row pointers iptr. */
lr_status lr_shard_rows(const int64_t* iptr, int32_t row_begin, int32_t row_end, int32_t world, int32_t* bounds);
/* The exchange schedule of one sharded unit: every rank's shard cut into
 * `chunks` nnz-balanced pieces of whole rows (world * chunks + 1 bounds; rank
 * q's chunk j = [cuts[q*chunks+j], cuts[q*chunks+j+1])).  Per iteration chunk j
 * is computed, then every rank's chunk j is broadcast (root order 0..world-1),
 * the last chunk followed by the all-reduce(max); LR_XCHG_CHUNKS sets
 * `chunks` (default 4). */
/* The rows of one level's units [unit_begin, unit_end) split over `world`
 * ranks for its CTA-solved units (world + 1 row bounds over the layout's
 * iptr / xptr / unit_row_begin / unit_kind): each rank solves the units
 * starting in its range (singleton groups and grid rows cut anywhere), the
 * ranges are then broadcast from their owners.  Applied to levels of at least
 * LR_DIST_MIN_ROWS rows (default 65536) when a communicator is set;
 * LR_DIST_LEVELS=0 replicates every level. */
lr_status lr_split_level_rows(const int64_t* iptr, const int64_t* xptr, const int32_t* unit_row_begin,
                              const uint8_t* unit_kind, int32_t unit_begin, int32_t unit_end, int32_t world,
                              int32_t* bounds);
lr_status lr_exchange_cuts(const int64_t* iptr, int32_t row_begin, int32_t row_end, int32_t world, int32_t chunks,
                           int32_t* cuts);

/* cudaStream_t the context launches on. */
void* lr_ctx_stream(lr_ctx* ctx);
/* UnitRecord::wall_ms (proj/src/engine.cpp:28,56) on the GPU: with
 * LR_UNIT_TIMES=1 set at upload, every level task and large-CAC CTA records
 * device timestamps, and after each solve ms[u] = the span from the first to
 * the last of unit u's tasks (units of one level run concurrently), plus its
 * grid SpMV time for a grid SccLarge unit.  LR_EINVAL when not enabled. */
lr_status lr_ctx_unit_times(const lr_ctx* ctx, double* ms, int64_t n_units);
/* Device bytes held by the context. */
int64_t lr_ctx_device_bytes(const lr_ctx* ctx);
/* Levels whose grid power series runs as K5 (k_spmv_blk: dest-row blocks,
   source-sorted in-edges, built at upload); no reference counterpart -- an
   introspection hook for tests and the bench. */
int32_t lr_ctx_blk_units(const lr_ctx* ctx);
void lr_ctx_free(lr_ctx* ctx);

/* ------------------------------------------------- one-call drop-in */
/* SolveReport (proj/include/levelrank/engine.hpp:30-67), scalar fields. */
typedef struct lr_report {
  int64_t vertices, edges, components, scc_components, cac_components, singleton_cacs;
  int32_t largest_component, largest_is_scc, max_level, level_count;
  int64_t large_scc_vertices;
  double eps_tot, eps_avg;
  int64_t total_iterations, iterative_edge_work, iterative_edges, single_pass_edge_work,
      cross_edge_count, total_edge_work;
  double mean_iterations_per_edge;
  int32_t all_weights_zero, threads;
  double wall_ms;
  int64_t n_units;
  double plan_ms;   /* host partition + layout */
  double upload_ms; /* H2D of the layout */
  double solve_ms;  /* lr_solve incl. weight H2D and rank D2H */
  double device_ms; /* device time of the level loop + normalisation */
} lr_report;

/* compute_pagerank (proj/src/engine.cpp:89-182; engine.hpp:92-95): partition,
 * layout, upload, device solve, report.  ranks (n) = R3, r1 (n, nullable).
 * unit_iters (nullable, capacity unit_cap). */
lr_status lr_compute_pagerank(const lr_graph* g, const double* w, int64_t wn, double c, double tol,
                              int32_t small_threshold, int device, double* ranks, double* r1,
                              lr_report* report, int64_t* unit_iters, int64_t unit_cap);

/* compute_baseline (proj/src/engine.cpp:184-218; engine.hpp:98-99): the
 * whole-graph power series on the GPU, report as the reference fills it
 * (total_iterations, iterative_edge_work = iterations * walk edges, ...). */
lr_status lr_compute_baseline(const lr_graph* g, const double* w, int64_t wn, double c, double tol,
                              int device, double* ranks, double* r1, lr_report* report);

/* --------------------------------------------------------- output formats */
/* The reference's writers, byte-compatible. */
typedef struct lr_unit_record { /* UnitRecord (engine.hpp:20-27) */
  int32_t kind;                 /* 0 singleton_group, 1 cac, 2 scc_small, 3 scc_large */
  int32_t level, size, reserved;
  int64_t edges, iterations;
  double wall_ms;
} lr_unit_record;
typedef struct lr_report_meta { /* the SolveReport fields lr_report does not carry */
  const char* method;           /* "partitioned" | "baseline" */
  const char* mode;             /* "sequential" | "parallel" */
  double c, tol;
  int32_t keep_loops, small_threshold, threads, reserved;
} lr_report_meta;
/* fmt 0: SolveReport::write_text (proj/src/report.cpp:24-60); 1: write_json
 * (:62-113); 2: one bench CSV row, 3: the bench CSV header (proj/src/cli.cpp:262-281).
 * *out is malloc'ed (release with lr_string_free), *len its length. */
lr_status lr_report_format(const lr_report* rep, const lr_report_meta* meta, const lr_unit_record* units,
                           int64_t n_units, int fmt, char** out, int64_t* len);
/* write_ranks (proj/src/cli.cpp:80-83): "v<TAB>rank" lines, 12 significant
 * digits; to a string, or straight to a file (path). */
lr_status lr_ranks_format(const double* ranks, int64_t n, char** out, int64_t* len);
lr_status lr_ranks_write(const double* ranks, int64_t n, const char* path);
void lr_string_free(char* s);

/* The unit solvers (proj/include/levelrank/solvers.hpp:31-54) on the GPU:
 * kind 0 solve_singletons, 1 solve_cac, 2 solve_small_scc, 3 solve_large_scc;
 * global_ids[m] the unit's vertices (local id = index), edge_src/dst[n_edges]
 * its intra edges in local ids, w_local[m] its start weights.  ranks_out[m];
 * iterations_out (kind 3) and edge_visits_out (kind 1) may be NULL. */
lr_status lr_solve_unit(const lr_graph* g, int kind, const int32_t* global_ids, int32_t m, const int32_t* edge_src,
                        const int32_t* edge_dst, int64_t n_edges, const double* w_local, double c, double tol,
                        int device, double* ranks_out, int64_t* iterations_out, int64_t* edge_visits_out);

/* solve_large_scc with PowerSeriesStats (solvers.cpp:128-162, solvers.hpp:23-27)
 * in its instrumented GPU form, on a unit given as a pull CSR (row i's in-edge
 * sources ascending; kept self-loops included), push factors pf = c/deg and
 * start weights w.  ranks[m]; *iterations; l1[k] = ||inc_k||_1 for the first
 * min(iterations, l1_cap) iterations; *min_entry = smallest increment entry.
 * LR_ENOCONV past `cap` iterations. */
lr_status lr_series_stats_csr(int device, int32_t m, const long long* ptr, const int32_t* src, const double* pf,
                              const double* w, double tol, int64_t cap, double* ranks, int64_t* iterations,
                              double* l1, int64_t l1_cap, double* min_entry);
/* The same from a unit of a graph (global ids, local edges), as solve_unit. */
lr_status lr_solve_large_scc_stats(const lr_graph* g, const int32_t* global_ids, int32_t m, const int32_t* edge_src,
                                   const int32_t* edge_dst, int64_t n_edges, const double* w_local, double c,
                                   double tol, int device, double* ranks_out, int64_t* iterations_out, double* l1,
                                   int64_t l1_cap, int64_t* l1_len, double* min_entry);

/* ------------------------------------------------------- solver helpers */
/* validate_params (proj/src/solvers.cpp:11-15). */
lr_status lr_validate_params(double c, double tol);
/* iteration_cap (proj/src/solvers.cpp:17-21). */
int64_t lr_iteration_cap(double c, double tol);
/* error_bound (proj/src/engine.cpp:74-81): out2 = {eps_tot, eps_avg}. */
void lr_error_bound(int64_t large_scc_vertices, int64_t vertex_count, double c, double tol,
                    double* out2);
/* propagate_weights (proj/src/engine.cpp:83-87) on the GPU: weights[dst] +=
 * c * ranks[src] / deg, summed per destination in input order. */
lr_status lr_propagate_weights(int device, const int32_t* src, const int32_t* dst,
                               const int32_t* deg, int64_t m, const double* ranks, int64_t n,
                               double c, double* weights);

/* ------------------------------------------------------ synthetic inputs */
/* Seeded, counter-based generators for the BASELINE.json configs (DESIGN.md
 * "Synthetic inputs").  Identical output for any thread count. */
lr_status lr_gen_rmat(int32_t scale, int64_t edge_factor, double a, double b, double c,
                      uint64_t seed, lr_graph** out);
/* Removes all out-edges of each vertex independently with probability p. */
lr_status lr_graph_dangle(const lr_graph* g, double p, uint64_t seed, lr_graph** out);
lr_status lr_gen_planted(int32_t n, int32_t n_scc, int32_t scc_min, int32_t scc_max,
                         int64_t scc_vertex_budget, double scc_out_degree, int64_t inter_edges,
                         double dangling_fraction, uint64_t seed, lr_graph** out);
lr_status lr_gen_deep_dag(int32_t levels, int32_t level_width, int32_t scc_min, int32_t scc_max,
                          double scc_out_degree, int32_t branch_min, int32_t branch_max,
                          double inter_out_degree, int32_t reach, uint64_t seed, lr_graph** out);

#ifdef __cplusplus
}
#endif
#endif
