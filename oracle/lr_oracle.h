/* TEST INFRASTRUCTURE ONLY -- the CPU checker for the level-scheduled
 * PageRank path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product
 * (paper_1609_09068_b200/) never links or calls it.
 *
 * A plain-C restatement of the reference algorithm (levelrank,
 * /root/reference/proj/src).  Every function cites the reference lines it
 * follows.  Parity pinned against (a) the reference's own known-answer tests
 * (tests/test_oracle_golden.py) and (b) the reference compiled from its own
 * sources (oracle/_ref, tests/golden/ fixtures made by tests/golden/make_golden.py).
 */
#ifndef LR_ORACLE_H
#define LR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { LRO_OK = 0, LRO_EINVAL = 1, LRO_ENOCONV = 2, LRO_ECYCLE = 3, LRO_EDEGEN = 4, LRO_ENOMEM = 7 };

typedef struct lro_graph lro_graph;
typedef struct lro_schedule lro_schedule;

/* Same field meanings as the reference SolveReport (engine.hpp:30-67). */
typedef struct {
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
} lro_report;

const char* lro_last_error(void);

/* Graph::from_edges (graph.cpp:14-36): sort, dedup, CSR, loop flags. */
int lro_graph_from_edges(int32_t n, const int32_t* src, const int32_t* dst, int64_t m, int keep,
                         lro_graph** out);
/* Borrow-free CSR constructor (rows must already be sorted and unique). */
int lro_graph_from_csr(int32_t n, const int64_t* off, const int32_t* tgt, int keep, lro_graph** out);
void lro_graph_free(lro_graph* g);
int64_t lro_graph_edges(const lro_graph* g);
void lro_graph_csr(const lro_graph* g, int64_t* off, int32_t* tgt, uint8_t* has_loop, int32_t* walk_deg);

/* find_components / find_components_scc_only (partition.cpp:52-145,246-250).
 * comp_of[n]; kinds/levels/sizes need capacity n; kinds: 0 = Scc, 1 = Cac.
 * stats3 = explore_edge_visits, merge_scan_edge_visits, finish_calls. */
int lro_find_components(const lro_graph* g, int merge_cacs, int32_t* comp_of, int32_t* kinds,
                        int32_t* levels, int32_t* sizes, int32_t* k_out, int32_t* max_level,
                        int64_t* stats3);

/* build_schedule (schedule.cpp:32-137) on the oracle's own partition. */
int lro_schedule_new(const lro_graph* g, int32_t small_threshold, lro_schedule** out);
void lro_schedule_free(lro_schedule* s);
/* [n_levels, n_units, n_ids, n_edges, n_cross, intra, cross, dropped] */
void lro_schedule_sizes(const lro_schedule* s, int64_t* out8);
void lro_schedule_get(const lro_schedule* s, int32_t* level_values, int32_t* level_unit_begin,
                      int64_t* level_cross_begin, int32_t* unit_kind, int32_t* unit_level,
                      int32_t* unit_size, int64_t* unit_ids_begin, int64_t* unit_edges_begin,
                      int32_t* ids, int32_t* edge_src, int32_t* edge_dst, int32_t* cross_src,
                      int32_t* cross_dst, int32_t* cross_deg, int32_t* permutation);

/* iteration_cap / error_bound (solvers.cpp:17-21, engine.cpp:74-81). */
int64_t lro_iteration_cap(double c, double tol);
void lro_error_bound(int64_t large, int64_t n, double c, double tol, double* out2);

/* compute_pagerank, Sequential (engine.cpp:89-182).  unit_iters/unit_kinds
 * (optional) receive per-unit iteration counts / kinds in schedule order. */
int lro_compute_pagerank(const lro_graph* g, const double* w, int64_t wn, double c, double tol,
                         int32_t small_threshold, double* ranks, lro_report* rep,
                         int64_t* unit_iters, int32_t* unit_kinds, int64_t unit_cap);
/* compute_baseline (engine.cpp:184-218 -> solvers.cpp:164-198). */
int lro_compute_baseline(const lro_graph* g, const double* w, int64_t wn, double c, double tol,
                         double* ranks, lro_report* rep);
/* R1 = R3 / ||R3||_1, the normalisation implied by oracle_r1_to_r3
 * (solvers.cpp:200-244): left-to-right fp64 sum, then one divide per entry. */
int lro_normalize_r1(const double* r3, int64_t n, double* r1);

/* Bounded CPU sample for bench.py's cpu_baseline: the large-SCC power series
 * (solvers.cpp:128-162, push COO scatter) of the schedule's largest SccLarge
 * unit, run for exactly `iters` multiplies from w.  Returns edge updates done
 * and wall ms. */
int lro_sample_large_scc(const lro_graph* g, const lro_schedule* s, const double* w, double c,
                         int64_t iters, int64_t* edge_updates, double* ms);

/* lr_gen.c: the BASELINE.json generators (same graphs as the product's
 * csrc/host/gen.cpp, asserted by tests/test_oracle_gen.py).  Edge lists are
 * malloc'ed; release them with lro_gen_free.  dangle_p > 0 applies config 3's
 * "each vertex loses all out-edges with probability p" (stream 2 of
 * dangle_seed) to the R-MAT edges. */
int lro_gen_rmat(int32_t scale, int64_t edge_factor, double a, double b, double c, uint64_t seed, double dangle_p,
                 uint64_t dangle_seed, int threads, int32_t** src, int32_t** dst, int64_t* m);
int lro_gen_planted(int32_t n, int32_t n_scc, int32_t smin, int32_t smax, int64_t budget, double out_degree,
                    int64_t inter_edges, double dangling_fraction, uint64_t seed, int32_t** src, int32_t** dst,
                    int64_t* m);
int lro_gen_deep_dag(int32_t levels, int32_t width, int32_t smin, int32_t smax, double scc_out_degree, int32_t bmin,
                     int32_t bmax, double inter_out_degree, int32_t reach, uint64_t seed, int threads, int32_t** src,
                     int32_t** dst, int64_t* m);
void lro_gen_free(int32_t* p);

#ifdef __cplusplus
}
#endif
#endif
