/* TEST INFRASTRUCTURE ONLY -- the BASELINE.json input generators, restated
 * in C for the CPU side of the measurement (bench.py --impl reference and the
 * cpu_baseline leg), so the reference arm never loads the product library.
 *
 * These are the repo's own generators (the reference has none for these
 * configs, SURVEY.md key finding 9): paper_1609_09068_b200/csrc/host/gen.cpp
 * is the product copy and tests/test_oracle_gen.py asserts that both give the
 * same graph.  Every random draw is splitmix64 addressed by (seed, stream,
 * index), so the output does not depend on the thread count.  Output is an
 * edge list (duplicates possible, self-loops possible except in R-MAT); the
 * caller builds the graph with the reference's own Graph::from_edges. */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "lr_oracle.h"

static uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static uint64_t draw(uint64_t seed, uint64_t stream, uint64_t i) {
  const uint64_t key = mix(seed * 0x9E3779B97F4A7C15ULL + (stream + 1) * 0xD1B54A32D192ED03ULL);
  return mix(key + (i + 1) * 0x9E3779B97F4A7C15ULL);
}
static double unit01(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }
static uint64_t below(uint64_t x, uint64_t n) { return (uint64_t)(((unsigned __int128)x * n) >> 64); }

typedef struct {
  int32_t *s, *d;
  int64_t n, cap;
} edges_t;

static int push(edges_t* e, int32_t u, int32_t v) {
  if (e->n == e->cap) {
    int64_t c = e->cap ? e->cap * 2 : 1024;
    int32_t* s = realloc(e->s, (size_t)c * 4);
    if (!s) return -1;
    e->s = s;
    int32_t* d = realloc(e->d, (size_t)c * 4);
    if (!d) return -1;
    e->d = d;
    e->cap = c;
  }
  e->s[e->n] = u;
  e->d[e->n] = v;
  e->n++;
  return 0;
}

void lro_gen_free(int32_t* p) { free(p); }

/* ------------------------------------------------------------------ R-MAT */
typedef struct {
  int32_t scale;
  uint64_t seed;
  uint32_t ta, tab, tabc;
  int per_edge;
  int64_t b0, b1;
  const double* drop_p; /* optional: drop edges of sources with unit01(draw(dseed,2,u)) < p */
  uint64_t dseed;
  edges_t out;
  int err;
} rmat_job;

static void* rmat_run(void* arg) {
  rmat_job* j = arg;
  for (int64_t i = j->b0; i < j->b1; ++i) {
    uint32_t su = 0, sv = 0;
    for (int l = 0; l < j->scale; ++l) {
      const uint64_t r = draw(j->seed, 1, (uint64_t)i * (uint64_t)j->per_edge + (uint64_t)(l / 2));
      const uint32_t x = (uint32_t)((l & 1) ? (r >> 32) : r);
      su = (su << 1) | (uint32_t)(x >= j->tab);
      sv = (sv << 1) | (uint32_t)((x >= j->ta && x < j->tab) || x >= j->tabc);
    }
    if (su == sv) continue;
    if (j->drop_p && unit01(draw(j->dseed, 2, su)) < *j->drop_p) continue;
    if (push(&j->out, (int32_t)su, (int32_t)sv)) {
      j->err = 1;
      return NULL;
    }
  }
  return NULL;
}

static uint32_t thresh(double x) {
  const double v = ldexp(x, 32);
  return (uint32_t)(v < 4294967295.0 ? v : 4294967295.0);
}

int lro_gen_rmat(int32_t scale, int64_t edge_factor, double a, double b, double c, uint64_t seed, double dangle_p,
                 uint64_t dangle_seed, int threads, int32_t** src, int32_t** dst, int64_t* m_out) {
  *src = *dst = NULL;
  *m_out = 0;
  if (scale < 1 || scale > 30 || edge_factor < 1 || threads < 1) return LRO_EINVAL;
  const int64_t m = edge_factor << scale;
  rmat_job* jobs = calloc((size_t)threads, sizeof *jobs);
  pthread_t* tid = calloc((size_t)threads, sizeof *tid);
  if (!jobs || !tid) return LRO_ENOMEM;
  for (int t = 0; t < threads; ++t) {
    rmat_job* j = &jobs[t];
    j->scale = scale;
    j->seed = seed;
    j->ta = thresh(a);
    j->tab = thresh(a + b);
    j->tabc = thresh(a + b + c);
    j->per_edge = (scale + 1) / 2;
    j->b0 = m * t / threads;
    j->b1 = m * (t + 1) / threads;
    j->drop_p = dangle_p > 0 ? &dangle_p : NULL;
    j->dseed = dangle_seed;
    pthread_create(&tid[t], NULL, rmat_run, j);
  }
  int64_t total = 0;
  int err = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    total += jobs[t].out.n;
    err |= jobs[t].err;
  }
  int32_t* S = err ? NULL : malloc((size_t)(total ? total : 1) * 4);
  int32_t* D = err ? NULL : malloc((size_t)(total ? total : 1) * 4);
  int64_t at = 0;
  for (int t = 0; t < threads; ++t) {
    if (S && D) {
      memcpy(S + at, jobs[t].out.s, (size_t)jobs[t].out.n * 4);
      memcpy(D + at, jobs[t].out.d, (size_t)jobs[t].out.n * 4);
    }
    at += jobs[t].out.n;
    free(jobs[t].out.s);
    free(jobs[t].out.d);
  }
  free(jobs);
  free(tid);
  if (!S || !D) {
    free(S);
    free(D);
    return LRO_ENOMEM;
  }
  *src = S;
  *dst = D;
  *m_out = total;
  return LRO_OK;
}

/* ------------------------------------------------------ planted (config 1) */
typedef struct {
  uint64_t seed, ctr;
} rng_t;
static uint64_t next(rng_t* r, uint64_t stream) { return draw(r->seed, stream, r->ctr++); }

int lro_gen_planted(int32_t n, int32_t n_scc, int32_t smin, int32_t smax, int64_t budget, double out_degree,
                    int64_t inter_edges, double dangling_fraction, uint64_t seed, int32_t** src, int32_t** dst,
                    int64_t* m_out) {
  *src = *dst = NULL;
  *m_out = 0;
  rng_t R = {seed, 0};
  int rc = LRO_ENOMEM;
  int64_t* size = calloc((size_t)n_scc + 1, sizeof *size);
  int32_t* perm = malloc((size_t)n * 4 + 4);
  int32_t* cb = malloc(((size_t)n + (size_t)n_scc + 2) * 4); /* component [cb[k], ce[k]) */
  int32_t* ce = malloc(((size_t)n + (size_t)n_scc + 2) * 4);
  uint8_t* has_out = calloc((size_t)n + 1, 1);
  uint8_t* dangling = calloc((size_t)n + 1, 1);
  int32_t* leaves = malloc((size_t)n * 4 + 4);
  int32_t *cidx = NULL, *at_index = NULL, *comp_of = NULL;
  edges_t E = {0};
  if (!size || !perm || !cb || !ce || !has_out || !dangling || !leaves) goto out;
  int64_t total = 0;
  for (int32_t k = 0; k < n_scc; ++k) {
    size[k] = smin + (int64_t)below(next(&R, 10), (uint64_t)(smax - smin + 1));
    total += size[k];
  }
  if (budget > 0 && total > budget)
    for (int32_t k = 0; k < n_scc; ++k) {
      const int64_t s = size[k] * budget / total;
      size[k] = s > smin ? s : smin;
    }
  total = 0;
  for (int32_t k = 0; k < n_scc; ++k) total += size[k];
  if (total > n) {
    rc = LRO_EINVAL;
    goto out;
  }
  for (int32_t i = 0; i < n; ++i) perm[i] = i;
  for (int32_t i = n - 1; i > 0; --i) {
    const int64_t j = (int64_t)below(next(&R, 11), (uint64_t)i + 1);
    const int32_t t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
#define EDGE(u, v) \
  if (push(&E, perm[(u)], perm[(v)])) goto out
  int64_t K = 0;
  int32_t at = 0;
  for (int32_t k = 0; k < n_scc; ++k) {
    const int32_t b = at;
    at += (int32_t)size[k];
    for (int32_t v = b; v < at; ++v) EDGE(v, v + 1 < at ? v + 1 : b);
    const double p = (out_degree - 1.0) / (double)(size[k] - 1);
    for (int32_t u = b; u < at; ++u)
      for (int32_t v = b; v < at; ++v)
        if (u != v && unit01(next(&R, 12)) < p) EDGE(u, v);
    cb[K] = b;
    ce[K] = at;
    ++K;
  }
  for (int32_t v = 0; v < at; ++v) has_out[v] = 1;
  int32_t root = at;
  for (int32_t v = at; v < n; ++v) {
    if (v == root || below(next(&R, 13), 16) == 0) {
      if (v != root) {
        cb[K] = root;
        ce[K] = v;
        ++K;
      }
      root = v;
      continue;
    }
    const int32_t parent = root + (int32_t)below(next(&R, 14), (uint64_t)(v - root));
    EDGE(parent, v);
    has_out[parent] = 1;
  }
  if (at < n) {
    cb[K] = root;
    ce[K] = n;
    ++K;
  }
  cidx = malloc((size_t)K * 4 + 4);
  at_index = malloc((size_t)K * 4 + 4);
  comp_of = malloc((size_t)n * 4 + 4);
  if (!cidx || !at_index || !comp_of) goto out;
  for (int64_t i = 0; i < K; ++i) cidx[i] = (int32_t)i;
  for (int64_t i = K - 1; i > 0; --i) {
    const int64_t j = (int64_t)below(next(&R, 15), (uint64_t)i + 1);
    const int32_t t = cidx[i];
    cidx[i] = cidx[j];
    cidx[j] = t;
  }
  for (int64_t k = 0; k < K; ++k) at_index[cidx[k]] = (int32_t)k;
  for (int64_t k = 0; k < K; ++k)
    for (int32_t v = cb[k]; v < ce[k]; ++v) comp_of[v] = (int32_t)k;
  int64_t nl = 0;
  for (int32_t v = 0; v < n; ++v)
    if (!has_out[v]) leaves[nl++] = v;
  for (int64_t i = nl; i > 1; --i) {
    const int64_t j = (int64_t)below(next(&R, 16), (uint64_t)i);
    const int32_t t = leaves[i - 1];
    leaves[i - 1] = leaves[j];
    leaves[j] = t;
  }
  const int64_t want = (int64_t)(dangling_fraction * n);
  const int64_t keep = nl < want ? nl : want;
  for (int64_t i = 0; i < keep; ++i) dangling[leaves[i]] = 1;
  int64_t used = 0;
  /* one inter-component edge from u to a uniform vertex of a later component */
#define INTER(u, ok)                                                                      \
  do {                                                                                    \
    const int32_t ci = cidx[comp_of[(u)]];                                                \
    (ok) = 0;                                                                             \
    if ((int64_t)ci + 1 < K) {                                                            \
      const int32_t cj = ci + 1 + (int32_t)below(next(&R, 17), (uint64_t)(K - ci - 1));  \
      const int32_t b = cb[at_index[cj]], e = ce[at_index[cj]];                           \
      EDGE((u), b + (int32_t)below(next(&R, 18), (uint64_t)(e - b)));                     \
      (ok) = 1;                                                                           \
    }                                                                                     \
  } while (0)
  for (int32_t v = 0; v < n && used < inter_edges; ++v)
    if (!has_out[v] && !dangling[v]) {
      int ok;
      INTER(v, ok);
      used += ok;
    }
  while (used < inter_edges) {
    const int32_t u = (int32_t)below(next(&R, 19), (uint64_t)n);
    if (dangling[u]) continue;
    int ok;
    INTER(u, ok);
    used += ok;
    if (K < 2) break;
  }
#undef INTER
#undef EDGE
  *src = E.s;
  *dst = E.d;
  *m_out = E.n;
  E.s = E.d = NULL;
  rc = LRO_OK;
out:
  free(E.s);
  free(E.d);
  free(size);
  free(perm);
  free(cb);
  free(ce);
  free(has_out);
  free(dangling);
  free(leaves);
  free(cidx);
  free(at_index);
  free(comp_of);
  return rc;
}

/* ----------------------------------------------------- deep DAG (config 4) */
typedef struct {
  int32_t levels, width, smin, smax, bmin, bmax, reach;
  double scc_out_degree, inter_out_degree;
  uint64_t seed;
  int32_t lv0, lv1;
  edges_t out;
  int err;
} dag_job;

static void* dag_run(void* arg) {
  dag_job* J = arg;
#define PUSH(u, v)                     \
  if (push(&J->out, (u), (v))) {       \
    J->err = 1;                        \
    return NULL;                       \
  }
  for (int32_t lv = J->lv0; lv < J->lv1; ++lv) {
    rng_t R = {J->seed, 0};
    const uint64_t sb = (uint64_t)lv * 64;
    const int32_t base = (int32_t)((int64_t)lv * J->width);
    int32_t at = 0;
    int scc = 1;
    while (at < J->width) {
      int32_t sz = J->smin + (int32_t)below(next(&R, sb + 1), (uint64_t)(J->smax - J->smin + 1));
      if (sz > J->width - at) sz = J->width - at;
      const int32_t b = base + at, e = b + sz;
      if (scc && sz >= 2) {
        for (int32_t v = b; v < e; ++v) PUSH(v, v + 1 < e ? v + 1 : b);
        const double extra = J->scc_out_degree - 1.0;
        for (int32_t v = b; v < e; ++v) {
          const int32_t k = (int32_t)extra + (unit01(next(&R, sb + 2)) < extra - floor(extra));
          for (int32_t j = 0; j < k; ++j) {
            int32_t w = b + (int32_t)below(next(&R, sb + 3), (uint64_t)(sz - 1));
            if (w >= v) ++w;
            PUSH(v, w);
          }
        }
      } else {
        int32_t filled = 1;
        for (int32_t i = 0; i < sz && filled < sz; ++i) {
          const int32_t kids = J->bmin + (int32_t)below(next(&R, sb + 4), (uint64_t)(J->bmax - J->bmin + 1));
          for (int32_t j = 0; j < kids && filled < sz; ++j, ++filled) PUSH(b + i, b + filled);
        }
      }
      at += sz;
      scc = !scc;
    }
    const double mean = J->inter_out_degree;
    for (int32_t v = base; v < base + J->width; ++v) {
      const int32_t k = (int32_t)mean + (unit01(next(&R, sb + 5)) < mean - floor(mean));
      for (int32_t j = 0; j < k; ++j) {
        const int32_t tl = lv + 1 + (int32_t)below(next(&R, sb + 6), (uint64_t)J->reach);
        if (tl >= J->levels) continue;
        PUSH(v, (int32_t)((int64_t)tl * J->width) + (int32_t)below(next(&R, sb + 7), (uint64_t)J->width));
      }
    }
  }
#undef PUSH
  return NULL;
}

int lro_gen_deep_dag(int32_t levels, int32_t width, int32_t smin, int32_t smax, double scc_out_degree, int32_t bmin,
                     int32_t bmax, double inter_out_degree, int32_t reach, uint64_t seed, int threads, int32_t** src,
                     int32_t** dst, int64_t* m_out) {
  *src = *dst = NULL;
  *m_out = 0;
  if ((int64_t)levels * width > 2147483646 || threads < 1) return LRO_EINVAL;
  dag_job* jobs = calloc((size_t)threads, sizeof *jobs);
  pthread_t* tid = calloc((size_t)threads, sizeof *tid);
  if (!jobs || !tid) return LRO_ENOMEM;
  for (int t = 0; t < threads; ++t) {
    dag_job* j = &jobs[t];
    *j = (dag_job){levels, width, smin, smax, bmin, bmax, reach, scc_out_degree, inter_out_degree, seed,
                   (int32_t)((int64_t)levels * t / threads), (int32_t)((int64_t)levels * (t + 1) / threads),
                   {0}, 0};
    pthread_create(&tid[t], NULL, dag_run, j);
  }
  int64_t total = 0;
  int err = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    total += jobs[t].out.n;
    err |= jobs[t].err;
  }
  int32_t* S = err ? NULL : malloc((size_t)(total ? total : 1) * 4);
  int32_t* D = err ? NULL : malloc((size_t)(total ? total : 1) * 4);
  int64_t at = 0;
  for (int t = 0; t < threads; ++t) {
    if (S && D) {
      memcpy(S + at, jobs[t].out.s, (size_t)jobs[t].out.n * 4);
      memcpy(D + at, jobs[t].out.d, (size_t)jobs[t].out.n * 4);
    }
    at += jobs[t].out.n;
    free(jobs[t].out.s);
    free(jobs[t].out.d);
  }
  free(jobs);
  free(tid);
  if (!S || !D) {
    free(S);
    free(D);
    return LRO_ENOMEM;
  }
  *src = S;
  *dst = D;
  *m_out = total;
  return LRO_OK;
}
