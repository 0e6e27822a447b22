/* TEST INFRASTRUCTURE ONLY -- CPU oracle (checker) for the level-scheduled
 * PageRank path; see lr_oracle.h.  Plain C restatement of the reference
 * levelrank algorithm (/root/reference/proj/src), function by function.
 * Scalar, single-threaded, and deliberately literal: every loop runs in the
 * same order as the reference so that all unit kinds except SccSmall (dense
 * LU) reproduce the reference's fp64 results bit for bit.
 */
#define _POSIX_C_SOURCE 200809L
#include "lr_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* lro_last_error(void) { return g_err; }

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec * 1e3 + (double)ts.tv_nsec * 1e-6;
}

#define XALLOC(ptr, count)                                                \
  do {                                                                    \
    size_t cnt_ = (size_t)(count);                                        \
    (ptr) = calloc(cnt_ ? cnt_ : 1, sizeof *(ptr));                       \
    if (!(ptr)) return fail(LRO_ENOMEM, "out of host memory");            \
  } while (0)

/* ------------------------------------------------------------------ graph */

struct lro_graph {
  int32_t n;
  int64_t m;
  int64_t* off;
  int32_t* tgt;
  uint8_t* loop;
  int keep;
};

/* Graph::walk_out_degree (graph.hpp:61-65). */
static int32_t walk_deg(const lro_graph* g, int32_t u) {
  int32_t d = (int32_t)(g->off[u + 1] - g->off[u]);
  if (!g->keep && g->loop[u]) --d;
  return d;
}

static void radix_sort_u64(uint64_t* a, uint64_t* tmp, int64_t m) {
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = pass * 16;
    int64_t* count = calloc(65537, sizeof *count);
    for (int64_t i = 0; i < m; ++i) ++count[((a[i] >> shift) & 0xffff) + 1];
    for (int b = 0; b < 65536; ++b) count[b + 1] += count[b];
    for (int64_t i = 0; i < m; ++i) tmp[count[(a[i] >> shift) & 0xffff]++] = a[i];
    memcpy(a, tmp, (size_t)m * sizeof *a);
    free(count);
  }
}

/* Graph::from_edges (graph.cpp:14-36): range check, sort, unique, CSR. */
int lro_graph_from_edges(int32_t n, const int32_t* src, const int32_t* dst, int64_t m, int keep,
                         lro_graph** out) {
  for (int64_t i = 0; i < m; ++i)
    if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n)
      return fail(LRO_EINVAL, "edge endpoint out of range");
  uint64_t *key, *tmp;
  XALLOC(key, m);
  XALLOC(tmp, m);
  for (int64_t i = 0; i < m; ++i) key[i] = ((uint64_t)(uint32_t)src[i] << 32) | (uint32_t)dst[i];
  radix_sort_u64(key, tmp, m);
  free(tmp);
  int64_t u = 0;
  for (int64_t i = 0; i < m; ++i)
    if (i == 0 || key[i] != key[i - 1]) key[u++] = key[i];
  lro_graph* g = calloc(1, sizeof *g);
  g->n = n;
  g->m = u;
  g->keep = keep;
  XALLOC(g->off, (int64_t)n + 1);
  XALLOC(g->tgt, u);
  XALLOC(g->loop, n);
  for (int64_t i = 0; i < u; ++i) ++g->off[(key[i] >> 32) + 1];
  for (int64_t i = 1; i <= n; ++i) g->off[i] += g->off[i - 1];
  for (int64_t i = 0; i < u; ++i) {
    const int32_t a = (int32_t)(key[i] >> 32), b = (int32_t)(uint32_t)key[i];
    g->tgt[i] = b;
    if (a == b) g->loop[a] = 1;
  }
  free(key);
  *out = g;
  return LRO_OK;
}

int lro_graph_from_csr(int32_t n, const int64_t* off, const int32_t* tgt, int keep, lro_graph** out) {
  lro_graph* g = calloc(1, sizeof *g);
  g->n = n;
  g->m = off[n];
  g->keep = keep;
  XALLOC(g->off, (int64_t)n + 1);
  XALLOC(g->tgt, g->m);
  XALLOC(g->loop, n);
  memcpy(g->off, off, ((size_t)n + 1) * sizeof *off);
  memcpy(g->tgt, tgt, (size_t)g->m * sizeof *tgt);
  for (int32_t a = 0; a < n; ++a)
    for (int64_t e = off[a]; e < off[a + 1]; ++e)
      if (tgt[e] == a) g->loop[a] = 1;
  *out = g;
  return LRO_OK;
}

void lro_graph_free(lro_graph* g) {
  if (!g) return;
  free(g->off);
  free(g->tgt);
  free(g->loop);
  free(g);
}

int64_t lro_graph_edges(const lro_graph* g) { return g->m; }

void lro_graph_csr(const lro_graph* g, int64_t* off, int32_t* tgt, uint8_t* has_loop, int32_t* wdeg) {
  memcpy(off, g->off, ((size_t)g->n + 1) * sizeof *off);
  memcpy(tgt, g->tgt, (size_t)g->m * sizeof *tgt);
  for (int32_t u = 0; u < g->n; ++u) {
    has_loop[u] = g->loop[u];
    wdeg[u] = walk_deg(g, u);
  }
}

/* ------------------------------------------------------------ union-find */
/* UnionFind (union_find.hpp:11-45): union by depth + path compression. */
typedef struct {
  int32_t* parent;
  int32_t* depth;
} uf_t;

static int32_t uf_find(uf_t* uf, int32_t x) {
  int32_t root = x;
  while (uf->parent[root] != root) root = uf->parent[root];
  while (uf->parent[x] != root) {
    const int32_t next = uf->parent[x];
    uf->parent[x] = root;
    x = next;
  }
  return root;
}

static void uf_unite(uf_t* uf, int32_t a, int32_t b) {
  a = uf_find(uf, a);
  b = uf_find(uf, b);
  if (a == b) return;
  if (uf->depth[a] < uf->depth[b]) {
    const int32_t t = a;
    a = b;
    b = t;
  }
  uf->parent[b] = a;
  if (uf->depth[a] == uf->depth[b]) ++uf->depth[a];
}

/* -------------------------------------------------------------- partition */

static int32_t imax(int32_t a, int32_t b) { return a > b ? a : b; }
static int32_t imin(int32_t a, int32_t b) { return a < b ? a : b; }

/* run_tarjan (partition.cpp:52-145) + assemble (partition.cpp:23-50). */
int lro_find_components(const lro_graph* g, int merge_cacs, int32_t* comp_of, int32_t* kinds,
                        int32_t* levels, int32_t* sizes, int32_t* k_out, int32_t* max_level,
                        int64_t* stats3) {
  const int32_t n = g->n;
  int32_t *order, *low, *level, *pending, *fr_v, *absorb, *id_of_root;
  int64_t* fr_cur;
  uint8_t *assigned, *is_scc;
  uf_t uf;
  XALLOC(order, n);
  XALLOC(low, n);
  XALLOC(level, n);
  XALLOC(pending, n);
  XALLOC(fr_v, n);
  XALLOC(fr_cur, n);
  XALLOC(absorb, n);
  XALLOC(id_of_root, n);
  XALLOC(assigned, n);
  XALLOC(is_scc, n);
  XALLOC(uf.parent, n);
  XALLOC(uf.depth, n);
  for (int32_t v = 0; v < n; ++v) {
    order[v] = -1;
    uf.parent[v] = v;
    uf.depth[v] = 1;
  }
  int64_t explore = 0, merge_scan = 0, finish_calls = 0;
  int32_t next_order = 0, np = 0, nf = 0;

  for (int32_t s = 0; s < n; ++s) {
    if (order[s] >= 0) continue;
    order[s] = low[s] = next_order++;
    level[s] = 1;
    pending[np++] = s;
    fr_v[nf] = s;
    fr_cur[nf++] = 0;
    while (nf > 0) {
      const int32_t v = fr_v[nf - 1];
      const int64_t deg = g->off[v + 1] - g->off[v];
      if (fr_cur[nf - 1] < deg) {
        const int32_t w = g->tgt[g->off[v] + fr_cur[nf - 1]++];
        ++explore;
        if (w == v) continue;
        if (order[w] < 0) {
          order[w] = low[w] = next_order++;
          level[w] = 1;
          pending[np++] = w;
          fr_v[nf] = w;
          fr_cur[nf++] = 0;
        } else if (assigned[w]) { /* update_from (partition.cpp:67-74) */
          level[v] = imax(level[v], level[w] + 1);
        } else {
          level[v] = imax(level[v], level[w]);
          low[v] = imin(low[v], low[w]);
        }
        continue;
      }
      --nf;
      /* finish (partition.cpp:76-113) */
      ++finish_calls;
      if (low[v] == order[v]) {
        int32_t first = np;
        while (pending[--first] != v) {
        }
        const int32_t members = np - first;
        for (int32_t i = first; i < np; ++i) {
          const int32_t mbr = pending[i];
          assigned[mbr] = 1;
          is_scc[mbr] = 1;
          level[mbr] = level[v];
          uf_unite(&uf, v, mbr);
        }
        np = first;
        if (members == 1) {
          is_scc[v] = 0;
          if (merge_cacs) {
            int32_t na = 0;
            int veto = 0;
            for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
              const int32_t w = g->tgt[e];
              ++merge_scan;
              if (w == v) continue;
              if (level[w] != level[v] - 1) continue;
              if (is_scc[w]) {
                veto = 1;
                break;
              }
              absorb[na++] = w;
            }
            if (!veto && na > 0) {
              --level[v];
              for (int32_t i = 0; i < na; ++i) uf_unite(&uf, v, absorb[i]);
            }
          }
        }
      }
      if (nf > 0) { /* update_from(parent, v) */
        const int32_t p = fr_v[nf - 1];
        if (assigned[v]) {
          level[p] = imax(level[p], level[v] + 1);
        } else {
          level[p] = imax(level[p], level[v]);
          low[p] = imin(low[p], low[v]);
        }
      }
    }
  }

  /* assemble: dense ids by first appearance, shift so min level is 0 */
  int32_t counter = 0;
  for (int32_t v = 0; v < n; ++v) id_of_root[v] = -1;
  for (int32_t v = 0; v < n; ++v) {
    const int32_t r = uf_find(&uf, v);
    if (id_of_root[r] < 0) {
      id_of_root[r] = counter;
      kinds[counter] = is_scc[r] ? 0 : 1;
      levels[counter] = level[r];
      sizes[counter] = 0;
      ++counter;
    }
    comp_of[v] = id_of_root[r];
    ++sizes[comp_of[v]];
  }
  int32_t mx = -1;
  if (counter > 0) {
    int32_t mn = levels[0];
    for (int32_t c = 1; c < counter; ++c) mn = imin(mn, levels[c]);
    for (int32_t c = 0; c < counter; ++c) {
      levels[c] -= mn;
      mx = imax(mx, levels[c]);
    }
  }
  *k_out = counter;
  *max_level = mx;
  if (stats3) {
    stats3[0] = explore;
    stats3[1] = merge_scan;
    stats3[2] = finish_calls;
  }
  free(order);
  free(low);
  free(level);
  free(pending);
  free(fr_v);
  free(fr_cur);
  free(absorb);
  free(id_of_root);
  free(assigned);
  free(is_scc);
  free(uf.parent);
  free(uf.depth);
  return LRO_OK;
}

/* --------------------------------------------------------------- schedule */

enum { KIND_SINGLETON = 0, KIND_CAC = 1, KIND_SCC_SMALL = 2, KIND_SCC_LARGE = 3 };

struct lro_schedule {
  int32_t n_levels;
  int32_t *level_values, *level_unit_begin;
  int64_t* level_cross_begin;
  int64_t n_units;
  int32_t *unit_kind, *unit_level, *unit_size;
  int64_t *unit_ids_begin, *unit_edges_begin;
  int32_t* ids;
  int32_t *edge_src, *edge_dst;
  int32_t *cross_src, *cross_dst, *cross_deg;
  int32_t* permutation;
  int64_t intra, cross, dropped;
  /* partition kept for the report census */
  int32_t k, max_level;
  int32_t *comp_of, *kinds, *levels, *sizes;
};

void lro_schedule_free(lro_schedule* s) {
  if (!s) return;
  free(s->level_values);
  free(s->level_unit_begin);
  free(s->level_cross_begin);
  free(s->unit_kind);
  free(s->unit_level);
  free(s->unit_size);
  free(s->unit_ids_begin);
  free(s->unit_edges_begin);
  free(s->ids);
  free(s->edge_src);
  free(s->edge_dst);
  free(s->cross_src);
  free(s->cross_dst);
  free(s->cross_deg);
  free(s->permutation);
  free(s->comp_of);
  free(s->kinds);
  free(s->levels);
  free(s->sizes);
  free(s);
}

/* sort_desc_by (schedule.cpp:14-28): stable counting sort, descending key. */
static void sort_desc_by(int32_t* items, int32_t count, const int32_t* key, int32_t max_key,
                         int32_t* scratch) {
  int64_t* cnt = calloc((size_t)max_key + 2, sizeof *cnt);
  for (int32_t i = 0; i < count; ++i) ++cnt[key[items[i]]];
  int64_t acc = 0;
  for (int32_t k = max_key; k >= 0; --k) {
    const int64_t c = cnt[k];
    cnt[k] = acc;
    acc += c;
  }
  for (int32_t i = 0; i < count; ++i) scratch[cnt[key[items[i]]]++] = items[i];
  memcpy(items, scratch, (size_t)count * sizeof *items);
  free(cnt);
}

/* build_schedule (schedule.cpp:32-137). */
int lro_schedule_new(const lro_graph* g, int32_t small_threshold, lro_schedule** out) {
  if (small_threshold < 1) return fail(LRO_EINVAL, "small_threshold must be at least 1");
  const int32_t n = g->n;
  lro_schedule* s = calloc(1, sizeof *s);
  XALLOC(s->comp_of, n);
  XALLOC(s->kinds, n);
  XALLOC(s->levels, n);
  XALLOC(s->sizes, n);
  int rc = lro_find_components(g, 1, s->comp_of, s->kinds, s->levels, s->sizes, &s->k,
                               &s->max_level, NULL);
  if (rc) return rc;
  const int32_t k = s->k;
  XALLOC(s->permutation, n);
  XALLOC(s->level_unit_begin, 1);
  XALLOC(s->level_cross_begin, 1);
  XALLOC(s->unit_ids_begin, 1);
  XALLOC(s->unit_edges_begin, 1);
  if (n == 0) {
    *out = s;
    return LRO_OK;
  }
  free(s->level_unit_begin);
  free(s->level_cross_begin);
  free(s->unit_ids_begin);
  free(s->unit_edges_begin);

  int32_t *comps, *scratch;
  XALLOC(comps, k);
  XALLOC(scratch, k);
  for (int32_t c = 0; c < k; ++c) comps[c] = c;
  sort_desc_by(comps, k, s->sizes, n, scratch);
  sort_desc_by(comps, k, s->levels, s->max_level, scratch);

  int32_t *mem_begin, *mem, *cursor;
  XALLOC(mem_begin, (int64_t)k + 1);
  XALLOC(mem, n);
  XALLOC(cursor, k);
  for (int32_t v = 0; v < n; ++v) ++mem_begin[s->comp_of[v] + 1];
  for (int32_t c = 0; c < k; ++c) mem_begin[c + 1] += mem_begin[c];
  for (int32_t c = 0; c < k; ++c) cursor[c] = mem_begin[c];
  for (int32_t v = 0; v < n; ++v) mem[cursor[s->comp_of[v]]++] = v;

  int32_t pos = 0;
  for (int32_t i = 0; i < k; ++i)
    for (int32_t j = mem_begin[comps[i]]; j < mem_begin[comps[i] + 1]; ++j) s->permutation[mem[j]] = pos++;

  s->n_levels = s->max_level + 1;
  XALLOC(s->level_values, s->n_levels);
  XALLOC(s->level_unit_begin, (int64_t)s->n_levels + 1);
  XALLOC(s->level_cross_begin, (int64_t)s->n_levels + 1);
  for (int32_t i = 0; i < s->n_levels; ++i) s->level_values[i] = s->max_level - i;

  /* units: at most k (one per multi-vertex comp) + one group per level */
  const int64_t ucap = (int64_t)k + s->n_levels;
  int32_t *ukind, *ulevel, *usize, *ucomp; /* ucomp = -1 for the singleton group */
  int32_t *unit_of_comp, *local_of, *singles;
  XALLOC(ukind, ucap);
  XALLOC(ulevel, ucap);
  XALLOC(usize, ucap);
  XALLOC(ucomp, ucap);
  XALLOC(unit_of_comp, k);
  XALLOC(local_of, n);
  XALLOC(singles, n);
  XALLOC(s->unit_ids_begin, ucap + 1);
  XALLOC(s->ids, n);
  int64_t nu = 0, nid = 0;
  int32_t walk = 0;
  while (walk < k) {
    const int32_t lvl = s->levels[comps[walk]];
    const int32_t li = s->max_level - lvl;
    s->level_unit_begin[li] = (int32_t)nu;
    const int64_t first_unit = nu;
    int32_t ns = 0;
    while (walk < k && s->levels[comps[walk]] == lvl) {
      const int32_t c = comps[walk++];
      if (s->sizes[c] == 1) {
        singles[ns++] = mem[mem_begin[c]];
        continue;
      }
      ukind[nu] = s->kinds[c] == 1 ? KIND_CAC
                  : s->sizes[c] < small_threshold ? KIND_SCC_SMALL
                                                  : KIND_SCC_LARGE;
      ulevel[nu] = lvl;
      usize[nu] = s->sizes[c];
      ucomp[nu] = c;
      ++nu;
    }
    if (ns > 0) {
      /* singles arrive in comp-id order, which is vertex order; sort anyway */
      for (int32_t i = 1; i < ns; ++i) {
        const int32_t x = singles[i];
        int32_t j = i - 1;
        if (singles[j] <= x) continue;
        while (j >= 0 && singles[j] > x) {
          singles[j + 1] = singles[j];
          --j;
        }
        singles[j + 1] = x;
      }
      int64_t slot = first_unit;
      while (slot < nu && usize[slot] >= ns) ++slot;
      for (int64_t u = nu; u > slot; --u) {
        ukind[u] = ukind[u - 1];
        ulevel[u] = ulevel[u - 1];
        usize[u] = usize[u - 1];
        ucomp[u] = ucomp[u - 1];
      }
      ukind[slot] = KIND_SINGLETON;
      ulevel[slot] = lvl;
      usize[slot] = ns;
      ucomp[slot] = -1;
      ++nu;
    }
    for (int64_t u = first_unit; u < nu; ++u) {
      s->unit_ids_begin[u] = nid;
      if (ucomp[u] >= 0) {
        const int32_t c = ucomp[u];
        unit_of_comp[c] = (int32_t)u;
        for (int32_t j = mem_begin[c]; j < mem_begin[c + 1]; ++j) {
          local_of[mem[j]] = (int32_t)(nid - s->unit_ids_begin[u]);
          s->ids[nid++] = mem[j];
        }
      } else {
        for (int32_t i = 0; i < ns; ++i) {
          unit_of_comp[s->comp_of[singles[i]]] = (int32_t)u;
          local_of[singles[i]] = i;
          s->ids[nid++] = singles[i];
        }
      }
    }
  }
  s->level_unit_begin[s->n_levels] = (int32_t)nu;
  /* levels with no components cannot exist (levels are longest paths), but
   * keep begin offsets monotone anyway */
  for (int32_t i = s->n_levels - 1; i >= 0; --i)
    if (s->level_unit_begin[i] > s->level_unit_begin[i + 1]) s->level_unit_begin[i] = s->level_unit_begin[i + 1];
  s->unit_ids_begin[nu] = nid;
  s->n_units = nu;
  s->unit_kind = ukind;
  s->unit_level = ulevel;
  s->unit_size = usize;

  /* edge split (schedule.cpp:112-135): count, then fill in generation order */
  int64_t *ecount, *xcount;
  XALLOC(ecount, nu + 1);
  XALLOC(xcount, (int64_t)s->n_levels + 1);
  for (int32_t u = 0; u < n; ++u) {
    const int32_t cu = s->comp_of[u];
    for (int64_t e = g->off[u]; e < g->off[u + 1]; ++e) {
      const int32_t v = g->tgt[e];
      if (u == v) {
        if (g->keep) {
          ++ecount[unit_of_comp[cu] + 1];
          ++s->intra;
        } else {
          ++s->dropped;
        }
        continue;
      }
      if (cu == s->comp_of[v]) {
        ++ecount[unit_of_comp[cu] + 1];
        ++s->intra;
      } else {
        ++xcount[s->max_level - s->levels[cu] + 1];
        ++s->cross;
      }
    }
  }
  for (int64_t u = 0; u < nu; ++u) ecount[u + 1] += ecount[u];
  for (int32_t l = 0; l < s->n_levels; ++l) xcount[l + 1] += xcount[l];
  XALLOC(s->unit_edges_begin, nu + 1);
  memcpy(s->unit_edges_begin, ecount, (size_t)(nu + 1) * sizeof *ecount);
  memcpy(s->level_cross_begin, xcount, ((size_t)s->n_levels + 1) * sizeof *xcount);
  XALLOC(s->edge_src, s->intra);
  XALLOC(s->edge_dst, s->intra);
  XALLOC(s->cross_src, s->cross);
  XALLOC(s->cross_dst, s->cross);
  XALLOC(s->cross_deg, s->cross);
  for (int32_t u = 0; u < n; ++u) {
    const int32_t cu = s->comp_of[u];
    for (int64_t e = g->off[u]; e < g->off[u + 1]; ++e) {
      const int32_t v = g->tgt[e];
      if (u == v && !g->keep) continue;
      if (cu == s->comp_of[v]) {
        const int64_t at = ecount[unit_of_comp[cu]]++;
        s->edge_src[at] = local_of[u];
        s->edge_dst[at] = local_of[v];
      } else {
        const int64_t at = xcount[s->max_level - s->levels[cu]]++;
        s->cross_src[at] = u;
        s->cross_dst[at] = v;
        s->cross_deg[at] = walk_deg(g, u);
      }
    }
  }
  free(ecount);
  free(xcount);
  free(comps);
  free(scratch);
  free(mem_begin);
  free(mem);
  free(cursor);
  free(ucomp);
  free(unit_of_comp);
  free(local_of);
  free(singles);
  *out = s;
  return LRO_OK;
}

void lro_schedule_sizes(const lro_schedule* s, int64_t* o) {
  o[0] = s->n_levels;
  o[1] = s->n_units;
  o[2] = s->n_units ? s->unit_ids_begin[s->n_units] : 0;
  o[3] = s->intra;
  o[4] = s->cross;
  o[5] = s->intra;
  o[6] = s->cross;
  o[7] = s->dropped;
}

void lro_schedule_get(const lro_schedule* s, int32_t* level_values, int32_t* level_unit_begin,
                      int64_t* level_cross_begin, int32_t* unit_kind, int32_t* unit_level,
                      int32_t* unit_size, int64_t* unit_ids_begin, int64_t* unit_edges_begin,
                      int32_t* ids, int32_t* edge_src, int32_t* edge_dst, int32_t* cross_src,
                      int32_t* cross_dst, int32_t* cross_deg, int32_t* permutation) {
  const size_t nl = (size_t)s->n_levels, nu = (size_t)s->n_units;
  if (nl) {
    memcpy(level_values, s->level_values, nl * 4);
    memcpy(level_unit_begin, s->level_unit_begin, (nl + 1) * 4);
    memcpy(level_cross_begin, s->level_cross_begin, (nl + 1) * 8);
  }
  if (nu) {
    memcpy(unit_kind, s->unit_kind, nu * 4);
    memcpy(unit_level, s->unit_level, nu * 4);
    memcpy(unit_size, s->unit_size, nu * 4);
    memcpy(unit_ids_begin, s->unit_ids_begin, (nu + 1) * 8);
    memcpy(unit_edges_begin, s->unit_edges_begin, (nu + 1) * 8);
    memcpy(ids, s->ids, (size_t)s->unit_ids_begin[nu] * 4);
  }
  memcpy(edge_src, s->edge_src, (size_t)s->intra * 4);
  memcpy(edge_dst, s->edge_dst, (size_t)s->intra * 4);
  memcpy(cross_src, s->cross_src, (size_t)s->cross * 4);
  memcpy(cross_dst, s->cross_dst, (size_t)s->cross * 4);
  memcpy(cross_deg, s->cross_deg, (size_t)s->cross * 4);
  for (int64_t v = 0; v < (int64_t)(s->n_units ? s->unit_ids_begin[nu] : 0); ++v) permutation[v] = s->permutation[v];
}

/* ---------------------------------------------------------------- solvers */

static int validate_params(double c, double tol) { /* solvers.cpp:11-15 */
  if (!(c > 0.0) || !(c < 1.0)) return fail(LRO_EINVAL, "continuation probability must lie in (0, 1)");
  if (!(tol > 0.0)) return fail(LRO_EINVAL, "tolerance must be positive");
  return LRO_OK;
}

int64_t lro_iteration_cap(double c, double tol) { /* solvers.cpp:17-21 */
  const double steps = log(tol) / log(c);
  const double capped = 10.0 * ceil(steps > 1.0 ? steps : 1.0);
  const int64_t cap = (int64_t)capped;
  return cap > 16 ? cap : 16;
}

void lro_error_bound(int64_t large, int64_t n, double c, double tol, double* out2) { /* engine.cpp:74-81 */
  out2[0] = (double)large * tol * c / (1.0 - c);
  out2[1] = n > 0 ? out2[0] / (double)n : 0.0;
}

typedef struct {
  const int32_t* ids;
  int32_t m;
  const int32_t* ea;
  const int32_t* eb;
  int64_t ne;
} unit_view;

/* solve_singletons (solvers.cpp:23-35) */
static void solve_singletons(const lro_graph* g, const unit_view* u, double* r, double c) {
  if (!g->keep) return;
  for (int32_t i = 0; i < u->m; ++i) {
    const int32_t v = u->ids[i];
    if (g->loop[v]) r[i] /= 1.0 - c / (double)walk_deg(g, v);
  }
}

/* solve_cac (solvers.cpp:37-88): Kahn queue, push shares rank*c/deg. */
static int solve_cac(const lro_graph* g, const unit_view* u, double* rank, double c) {
  const int32_t m = u->m;
  int32_t *offset, *target, *indeg, *queue, *cur;
  XALLOC(offset, (int64_t)m + 1);
  XALLOC(target, u->ne);
  XALLOC(indeg, m);
  XALLOC(queue, m);
  XALLOC(cur, m);
  for (int64_t e = 0; e < u->ne; ++e) {
    if (u->ea[e] == u->eb[e]) continue;
    ++offset[u->ea[e] + 1];
    ++indeg[u->eb[e]];
  }
  for (int32_t i = 0; i < m; ++i) offset[i + 1] += offset[i];
  for (int32_t i = 0; i < m; ++i) cur[i] = offset[i];
  for (int64_t e = 0; e < u->ne; ++e) {
    if (u->ea[e] == u->eb[e]) continue;
    target[cur[u->ea[e]]++] = u->eb[e];
  }
  int32_t qn = 0, head = 0;
  for (int32_t i = 0; i < m; ++i)
    if (indeg[i] == 0) queue[qn++] = i;
  while (head < qn) {
    const int32_t a = queue[head++];
    const int32_t ga = u->ids[a];
    if (g->keep && g->loop[ga]) rank[a] /= 1.0 - c / (double)walk_deg(g, ga);
    if (offset[a] == offset[a + 1]) continue;
    const double share = rank[a] * c / (double)walk_deg(g, ga);
    for (int32_t e = offset[a]; e < offset[a + 1]; ++e) {
      const int32_t b = target[e];
      rank[b] += share;
      if (--indeg[b] == 0) queue[qn++] = b;
    }
  }
  free(offset);
  free(target);
  free(indeg);
  free(queue);
  free(cur);
  if (qn != m) return fail(LRO_ECYCLE, "cycle inside an acyclic component");
  return LRO_OK;
}

/* solve_small_scc -> solve_dense_system (solvers.cpp:92-116): dense
 * (I - cA^T) r = w, Gaussian elimination with partial pivoting (the
 * elimination order of test_support.cpp:75-111), residual check. */
static int solve_small_scc(const lro_graph* g, const unit_view* u, const double* w, double* r, double c) {
  const int32_t m = u->m;
  double *sys, *a, *rhs;
  XALLOC(sys, (int64_t)m * m);
  XALLOC(a, (int64_t)m * m);
  XALLOC(rhs, m);
  for (int32_t i = 0; i < m; ++i) sys[(int64_t)i * m + i] = 1.0;
  for (int64_t e = 0; e < u->ne; ++e) {
    const int32_t ea = u->ea[e], eb = u->eb[e];
    if (ea == eb && !g->keep) continue;
    sys[(int64_t)eb * m + ea] -= c / (double)walk_deg(g, u->ids[ea]);
  }
  memcpy(a, sys, (size_t)m * m * sizeof *a);
  memcpy(rhs, w, (size_t)m * sizeof *rhs);
  for (int32_t col = 0; col < m; ++col) {
    int32_t piv = col;
    for (int32_t row = col + 1; row < m; ++row)
      if (fabs(a[(int64_t)row * m + col]) > fabs(a[(int64_t)piv * m + col])) piv = row;
    if (piv != col) {
      for (int32_t j = 0; j < m; ++j) {
        const double t = a[(int64_t)col * m + j];
        a[(int64_t)col * m + j] = a[(int64_t)piv * m + j];
        a[(int64_t)piv * m + j] = t;
      }
      const double t = rhs[col];
      rhs[col] = rhs[piv];
      rhs[piv] = t;
    }
    const double d = a[(int64_t)col * m + col];
    if (d == 0.0) continue;
    for (int32_t row = col + 1; row < m; ++row) {
      const double f = a[(int64_t)row * m + col] / d;
      if (f == 0.0) continue;
      for (int32_t j = col; j < m; ++j) a[(int64_t)row * m + j] -= f * a[(int64_t)col * m + j];
      rhs[row] -= f * rhs[col];
    }
  }
  for (int32_t row = m - 1; row >= 0; --row) {
    double acc = rhs[row];
    for (int32_t j = row + 1; j < m; ++j) acc -= a[(int64_t)row * m + j] * r[j];
    r[row] = acc / a[(int64_t)row * m + row];
  }
  double residual = 0.0, wmax = 0.0, rmax = 0.0;
  for (int32_t i = 0; i < m; ++i) {
    double acc = 0.0;
    for (int32_t j = 0; j < m; ++j) acc += sys[(int64_t)i * m + j] * r[j];
    const double d = fabs(acc - w[i]);
    if (!(d <= residual)) residual = d; /* NaN-propagating max */
    if (fabs(w[i]) > wmax) wmax = fabs(w[i]);
    if (fabs(r[i]) > rmax) rmax = fabs(r[i]);
  }
  free(sys);
  free(a);
  free(rhs);
  if (!(residual <= 1e-8 * (1.0 + wmax + rmax))) return fail(LRO_EDEGEN, "dense solve degenerated numerically");
  return LRO_OK;
}

/* solve_large_scc (solvers.cpp:128-162): accumulated power series with a
 * push COO scatter, stop when max|inc| < tol, throw past the cap. */
static int solve_large_scc(const lro_graph* g, const unit_view* u, const double* w, double* rank,
                           double c, double tol, int64_t* iterations) {
  const int32_t m = u->m;
  *iterations = 0;
  if (m == 0) return LRO_OK;
  double *pf, *inc, *next;
  XALLOC(pf, m);
  XALLOC(inc, m);
  XALLOC(next, m);
  for (int32_t i = 0; i < m; ++i) pf[i] = c / (double)walk_deg(g, u->ids[i]);
  for (int32_t i = 0; i < m; ++i) rank[i] = inc[i] = w[i];
  const int64_t cap = lro_iteration_cap(c, tol);
  int rc = LRO_OK;
  double mx;
  do {
    memset(next, 0, (size_t)m * sizeof *next);
    for (int64_t e = 0; e < u->ne; ++e) {
      const int32_t a = u->ea[e], b = u->eb[e];
      if (a == b && !g->keep) continue;
      next[b] += pf[a] * inc[a];
    }
    double* t = inc;
    inc = next;
    next = t;
    for (int32_t i = 0; i < m; ++i) rank[i] += inc[i];
    ++*iterations;
    if (*iterations > cap) {
      rc = fail(LRO_ENOCONV, "power series failed to converge");
      break;
    }
    mx = fabs(inc[0]);
    for (int32_t i = 1; i < m; ++i)
      if (fabs(inc[i]) > mx) mx = fabs(inc[i]);
  } while (mx >= tol);
  free(pf);
  free(inc);
  free(next);
  return rc;
}

/* ----------------------------------------------------------------- engine */

static void fill_census(const lro_schedule* s, lro_report* rep) { /* partition.cpp:353-382 */
  rep->components = s->k;
  int32_t largest = 0;
  int32_t largest_scc = 0;
  for (int32_t i = 0; i < s->k; ++i) {
    if (s->kinds[i] == 0) {
      ++rep->scc_components;
    } else {
      ++rep->cac_components;
      if (s->sizes[i] == 1) ++rep->singleton_cacs;
    }
    if (s->sizes[i] > largest) {
      largest = s->sizes[i];
      largest_scc = s->kinds[i] == 0;
    }
  }
  rep->largest_component = largest;
  rep->largest_is_scc = largest_scc;
  rep->max_level = s->max_level;
  rep->level_count = s->max_level + 1;
}

/* compute_pagerank, Sequential (engine.cpp:89-182). */
int lro_compute_pagerank(const lro_graph* g, const double* w, int64_t wn, double c, double tol,
                         int32_t small_threshold, double* ranks, lro_report* rep,
                         int64_t* unit_iters, int32_t* unit_kinds, int64_t unit_cap) {
  int rc = validate_params(c, tol);
  if (rc) return rc;
  const int32_t n = g->n;
  if (wn != n) return fail(LRO_EINVAL, "weight vector does not match the vertex count");
  for (int32_t v = 0; v < n; ++v)
    if (w[v] < 0.0) return fail(LRO_EINVAL, "weights must be non-negative");
  const double t0 = now_ms();
  lro_report local;
  memset(&local, 0, sizeof local);
  if (!rep) rep = &local;
  memset(rep, 0, sizeof *rep);
  rep->vertices = n;
  rep->edges = g->m;
  rep->max_level = -1;
  rep->threads = 1;
  for (int32_t v = 0; v < n; ++v) ranks[v] = 0.0;
  if (n == 0) return LRO_OK;
  double wmax = w[0];
  for (int32_t v = 1; v < n; ++v)
    if (w[v] > wmax) wmax = w[v];
  rep->all_weights_zero = wmax == 0.0;

  lro_schedule* s = NULL;
  rc = lro_schedule_new(g, small_threshold, &s);
  if (rc) return rc;
  fill_census(s, rep);

  double *work_w, *wl, *rl;
  XALLOC(work_w, n);
  XALLOC(wl, n);
  XALLOC(rl, n);
  memcpy(work_w, w, (size_t)n * sizeof *w);
  for (int32_t li = 0; li < s->n_levels && rc == LRO_OK; ++li) {
    for (int64_t ui = s->level_unit_begin[li]; ui < s->level_unit_begin[li + 1]; ++ui) {
      unit_view u;
      u.ids = s->ids + s->unit_ids_begin[ui];
      u.m = (int32_t)(s->unit_ids_begin[ui + 1] - s->unit_ids_begin[ui]);
      u.ea = s->edge_src + s->unit_edges_begin[ui];
      u.eb = s->edge_dst + s->unit_edges_begin[ui];
      u.ne = s->unit_edges_begin[ui + 1] - s->unit_edges_begin[ui];
      for (int32_t i = 0; i < u.m; ++i) wl[i] = work_w[u.ids[i]];
      int64_t it = 0;
      switch (s->unit_kind[ui]) {
        case KIND_SINGLETON:
          memcpy(rl, wl, (size_t)u.m * sizeof *rl);
          solve_singletons(g, &u, rl, c);
          break;
        case KIND_CAC:
          memcpy(rl, wl, (size_t)u.m * sizeof *rl);
          rc = solve_cac(g, &u, rl, c);
          break;
        case KIND_SCC_SMALL:
          rc = solve_small_scc(g, &u, wl, rl, c);
          break;
        default:
          rc = solve_large_scc(g, &u, wl, rl, c, tol, &it);
          break;
      }
      if (rc) break;
      for (int32_t i = 0; i < u.m; ++i) ranks[u.ids[i]] = rl[i];
      if (unit_iters && ui < unit_cap) unit_iters[ui] = it;
      if (unit_kinds && ui < unit_cap) unit_kinds[ui] = s->unit_kind[ui];
      rep->total_iterations += it;
      if (s->unit_kind[ui] == KIND_SCC_LARGE) {
        rep->iterative_edge_work += it * u.ne;
        rep->iterative_edges += u.ne;
        rep->large_scc_vertices += u.m;
      } else {
        rep->single_pass_edge_work += u.ne;
      }
    }
    if (rc) break;
    /* propagate_weights (engine.cpp:83-87) */
    for (int64_t e = s->level_cross_begin[li]; e < s->level_cross_begin[li + 1]; ++e)
      work_w[s->cross_dst[e]] += c * ranks[s->cross_src[e]] / (double)s->cross_deg[e];
  }
  rep->n_units = s->n_units;
  rep->cross_edge_count = s->cross;
  rep->single_pass_edge_work += s->cross;
  rep->total_edge_work = rep->iterative_edge_work + rep->single_pass_edge_work;
  rep->mean_iterations_per_edge =
      rep->iterative_edges > 0 ? (double)rep->iterative_edge_work / (double)rep->iterative_edges : 0.0;
  double eb[2];
  lro_error_bound(rep->large_scc_vertices, n, c, tol, eb);
  rep->eps_tot = eb[0];
  rep->eps_avg = eb[1];
  rep->wall_ms = now_ms() - t0;
  free(work_w);
  free(wl);
  free(rl);
  lro_schedule_free(s);
  return rc;
}

/* compute_baseline (engine.cpp:184-218) -> solve_baseline (solvers.cpp:164-198). */
int lro_compute_baseline(const lro_graph* g, const double* w, int64_t wn, double c, double tol,
                         double* ranks, lro_report* rep) {
  int rc = validate_params(c, tol);
  if (rc) return rc;
  const int32_t n = g->n;
  if (wn != n) return fail(LRO_EINVAL, "weight vector does not match the vertex count");
  for (int32_t v = 0; v < n; ++v)
    if (w[v] < 0.0) return fail(LRO_EINVAL, "weights must be non-negative");
  const double t0 = now_ms();
  lro_report local;
  if (!rep) rep = &local;
  memset(rep, 0, sizeof *rep);
  rep->vertices = n;
  rep->edges = g->m;
  rep->max_level = -1;
  rep->threads = 1;
  if (n == 0) return LRO_OK;
  double wmax = w[0];
  for (int32_t v = 1; v < n; ++v)
    if (w[v] > wmax) wmax = w[v];
  rep->all_weights_zero = wmax == 0.0;
  double *pf, *inc, *next;
  XALLOC(pf, n);
  XALLOC(inc, n);
  XALLOC(next, n);
  int64_t walk_edges = 0;
  for (int32_t u = 0; u < n; ++u) {
    const int32_t d = walk_deg(g, u);
    walk_edges += d;
    if (d > 0) pf[u] = c / (double)d;
  }
  for (int32_t u = 0; u < n; ++u) ranks[u] = inc[u] = w[u];
  const int64_t cap = lro_iteration_cap(c, tol);
  int64_t it = 0;
  double mx;
  do {
    memset(next, 0, (size_t)n * sizeof *next);
    for (int32_t u = 0; u < n; ++u) {
      if (inc[u] == 0.0) continue;
      const double push = pf[u] * inc[u];
      for (int64_t e = g->off[u]; e < g->off[u + 1]; ++e) {
        const int32_t v = g->tgt[e];
        if (u == v && !g->keep) continue;
        next[v] += push;
      }
    }
    double* t = inc;
    inc = next;
    next = t;
    for (int32_t u = 0; u < n; ++u) ranks[u] += inc[u];
    ++it;
    if (it > cap) {
      rc = fail(LRO_ENOCONV, "power series failed to converge");
      break;
    }
    mx = fabs(inc[0]);
    for (int32_t u = 1; u < n; ++u)
      if (fabs(inc[u]) > mx) mx = fabs(inc[u]);
  } while (mx >= tol);
  rep->total_iterations = it;
  rep->iterative_edge_work = it * walk_edges;
  rep->iterative_edges = walk_edges;
  rep->total_edge_work = rep->iterative_edge_work;
  rep->mean_iterations_per_edge = (double)it;
  rep->wall_ms = now_ms() - t0;
  free(pf);
  free(inc);
  free(next);
  return rc;
}

int lro_normalize_r1(const double* r3, int64_t n, double* r1) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += r3[i];
  if (!(s > 0.0)) {
    for (int64_t i = 0; i < n; ++i) r1[i] = 0.0;
    return fail(LRO_EINVAL, "start weights must carry positive mass");
  }
  for (int64_t i = 0; i < n; ++i) r1[i] = r3[i] / s;
  return LRO_OK;
}

int lro_sample_large_scc(const lro_graph* g, const lro_schedule* s, const double* w, double c,
                         int64_t iters, int64_t* edge_updates, double* ms) {
  int64_t best = -1, best_e = -1;
  for (int64_t u = 0; u < s->n_units; ++u) {
    const int64_t e = s->unit_edges_begin[u + 1] - s->unit_edges_begin[u];
    if (s->unit_kind[u] == KIND_SCC_LARGE && e > best_e) {
      best = u;
      best_e = e;
    }
  }
  *edge_updates = 0;
  *ms = 0.0;
  if (best < 0) return LRO_OK;
  const int32_t* ids = s->ids + s->unit_ids_begin[best];
  const int32_t m = (int32_t)(s->unit_ids_begin[best + 1] - s->unit_ids_begin[best]);
  const int32_t* ea = s->edge_src + s->unit_edges_begin[best];
  const int32_t* eb = s->edge_dst + s->unit_edges_begin[best];
  double *pf, *inc, *next, *rank;
  XALLOC(pf, m);
  XALLOC(inc, m);
  XALLOC(next, m);
  XALLOC(rank, m);
  for (int32_t i = 0; i < m; ++i) {
    pf[i] = c / (double)walk_deg(g, ids[i]);
    rank[i] = inc[i] = w[ids[i]];
  }
  const double t0 = now_ms();
  for (int64_t k = 0; k < iters; ++k) {
    memset(next, 0, (size_t)m * sizeof *next);
    for (int64_t e = 0; e < best_e; ++e) {
      if (ea[e] == eb[e] && !g->keep) continue;
      next[eb[e]] += pf[ea[e]] * inc[ea[e]];
    }
    double* t = inc;
    inc = next;
    next = t;
    double mx = 0.0;
    for (int32_t i = 0; i < m; ++i) {
      rank[i] += inc[i];
      if (fabs(inc[i]) > mx) mx = fabs(inc[i]);
    }
    (void)mx;
  }
  *ms = now_ms() - t0;
  *edge_updates = iters * best_e;
  free(pf);
  free(inc);
  free(next);
  free(rank);
  return LRO_OK;
}
