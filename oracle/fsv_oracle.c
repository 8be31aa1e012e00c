/*
 * fsv_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker, never the
 * product). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * / --impl reference legs may load this library.
 *
 * Plain-C restatement of the reference `svcc` CPU algorithms for the FastSV
 * hot path, in int32 vertex ids / int64 offsets, single-threaded and written
 * to be obviously correct:
 *
 *   oracle_uf_labels      union-find by rank with path compression followed
 *                         by a min-relabel pass scanning ids ascending
 *                         (/root/reference/pkg/src/svcc/oracle.py:12-55).
 *   oracle_fastsv_csr     all-flags FastSV, one commit per iteration,
 *                         edge-parallel form (algorithms.py:79-91) driven by
 *                         the gf-stability loop of _drive (algorithms.py:117-142).
 *   oracle_fastsv_la_csr  the same iteration in the matrix formulation of
 *                         fastsv_la (driver.py:64-120): persistent mngf
 *                         accumulator, scatter-min through the index snapshot,
 *                         two element-wise mins, gf extraction, termination on
 *                         count_diff(dup, gf) == 0.
 *   oracle_fastsv_edges   oracle_fastsv_csr over a raw pair list (both
 *                         orientations, self-loops and duplicates kept; the
 *                         E3 equivalence of SURVEY.md §8a).
 *
 * Parity of this file with the reference is pinned by tests/test_oracle.py
 * against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_INPUT 1
#define ORC_ERR_INVARIANT 3
#define ORC_ERR_NOMEM 5

/* ---- union-find (oracle.py:12-55) ------------------------------------- */

static int32_t uf_find(int32_t* parent, int32_t x) {
  int32_t root = x;
  while (parent[root] != root) root = parent[root];
  while (parent[x] != root) { /* path compression */
    int32_t next = parent[x];
    parent[x] = root;
    x = next;
  }
  return root;
}

int oracle_uf_labels(int64_t n, int64_t m, const int32_t* pairs, int32_t* labels) {
  if (n < 0) return ORC_ERR_INPUT;
  int32_t* parent = (int32_t*)malloc((size_t)(n ? n : 1) * sizeof(int32_t));
  uint8_t* rank = (uint8_t*)calloc((size_t)(n ? n : 1), 1);
  int32_t* smallest = (int32_t*)malloc((size_t)(n ? n : 1) * sizeof(int32_t));
  if (!parent || !rank || !smallest) { free(parent); free(rank); free(smallest); return ORC_ERR_NOMEM; }
  for (int64_t i = 0; i < n; ++i) { parent[i] = (int32_t)i; smallest[i] = -1; }
  for (int64_t e = 0; e < m; ++e) {
    int32_t a = pairs[2 * e], b = pairs[2 * e + 1];
    if (a < 0 || a >= n || b < 0 || b >= n) { free(parent); free(rank); free(smallest); return ORC_ERR_INPUT; }
    int32_t ra = uf_find(parent, a), rb = uf_find(parent, b);
    if (ra == rb) continue;
    if (rank[ra] < rank[rb]) { int32_t t = ra; ra = rb; rb = t; }
    parent[rb] = ra;
    if (rank[ra] == rank[rb]) rank[ra]++;
  }
  /* ids ascending: the first id seen in a class is its minimum */
  for (int64_t u = 0; u < n; ++u) {
    int32_t r = uf_find(parent, (int32_t)u);
    if (smallest[r] < 0) smallest[r] = (int32_t)u;
    labels[u] = smallest[r];
  }
  free(parent); free(rank); free(smallest);
  return ORC_OK;
}

/* ---- shared driver state ------------------------------------------------ */

typedef struct {
  int64_t n;
  int32_t *f, *fn, *gf, *gf_prev;
} orc_state;

static int state_init(orc_state* s, int64_t n) {
  size_t bytes = (size_t)(n ? n : 1) * sizeof(int32_t);
  s->n = n;
  s->f = (int32_t*)malloc(bytes); s->fn = (int32_t*)malloc(bytes);
  s->gf = (int32_t*)malloc(bytes); s->gf_prev = (int32_t*)malloc(bytes);
  if (!s->f || !s->fn || !s->gf || !s->gf_prev) return ORC_ERR_NOMEM;
  for (int64_t i = 0; i < n; ++i) s->f[i] = s->gf_prev[i] = (int32_t)i;
  return ORC_OK;
}

static void state_free(orc_state* s) { free(s->f); free(s->fn); free(s->gf); free(s->gf_prev); }

/* After fn is committed: count changes, record trace, rotate.
 * Returns 1 when the gf-stability stop rule fires (algorithms.py:139). */
static int finish_iteration(orc_state* s, int64_t it, int64_t cap, int64_t* gf_changed,
                            int64_t* f_changed, int32_t* snapshots, int* err) {
  int64_t n = s->n, gfc = 0, fc = 0;
  for (int64_t u = 0; u < n; ++u) {
    if (s->fn[u] > s->f[u]) *err = ORC_ERR_INVARIANT; /* _check_commit, algorithms.py:60-63 */
    fc += s->fn[u] != s->f[u];
  }
  for (int64_t u = 0; u < n; ++u) {
    int32_t g = s->fn[s->fn[u]];
    gfc += g != s->gf_prev[u];
    s->gf_prev[u] = g;
  }
  if (it < cap) {
    if (gf_changed) gf_changed[it] = gfc;
    if (f_changed) f_changed[it] = fc;
    if (snapshots) memcpy(snapshots + it * n, s->fn, (size_t)n * sizeof(int32_t));
  }
  int32_t* t = s->f; s->f = s->fn; s->fn = t;
  return gfc == 0;
}

static int finish_labels(orc_state* s, int32_t* labels) {
  /* labeling_from_parents star check (graph.py:116-117) */
  for (int64_t u = 0; u < s->n; ++u)
    if (s->f[s->f[u]] != s->f[u]) return ORC_ERR_INVARIANT;
  if (labels) memcpy(labels, s->f, (size_t)s->n * sizeof(int32_t));
  return ORC_OK;
}

/* ---- FastSV, edge-parallel form (algorithms.py:79-91, all flags) -------- */

int oracle_fastsv_csr(int64_t n, const int64_t* offsets, const int32_t* cols,
                      int64_t cap, int32_t* labels, int64_t* iterations,
                      int64_t* gf_changed, int64_t* f_changed, int32_t* snapshots) {
  orc_state s;
  int err = state_init(&s, n);
  if (err) { state_free(&s); return err; }
  int64_t it = 0;
  for (;;) {
    for (int64_t u = 0; u < n; ++u) s.gf[u] = s.f[s.f[u]];          /* gf = f[f] */
    memcpy(s.fn, s.f, (size_t)n * sizeof(int32_t));                 /* fn = f.copy() */
    for (int64_t u = 0; u < n; ++u) {
      int32_t fu = s.f[u];
      for (int64_t e = offsets[u]; e < offsets[u + 1]; ++e) {
        int32_t hv = s.gf[cols[e]];                                 /* hook_vals = gf[cols] */
        if (hv < s.fn[fu]) s.fn[fu] = hv;                           /* stochastic: fn[f[u]] <-min */
        if (hv < s.fn[u]) s.fn[u] = hv;                             /* aggressive: fn[u] <-min */
      }
    }
    for (int64_t u = 0; u < n; ++u) if (s.gf[u] < s.fn[u]) s.fn[u] = s.gf[u]; /* shortcut */
    int stop = finish_iteration(&s, it, cap, gf_changed, f_changed, snapshots, &err);
    ++it;
    if (err) break;
    if (stop) break;
  }
  if (!err) err = finish_labels(&s, labels);
  if (iterations) *iterations = it;
  state_free(&s);
  return err;
}

/* ---- same over a raw pair list (E3: self-loops/duplicates harmless) ----- */

int oracle_fastsv_edges(int64_t n, int64_t m, const int32_t* pairs,
                        int64_t cap, int32_t* labels, int64_t* iterations,
                        int64_t* gf_changed, int64_t* f_changed, int32_t* snapshots) {
  for (int64_t e = 0; e < 2 * m; ++e) if (pairs[e] < 0 || pairs[e] >= n) return ORC_ERR_INPUT;
  orc_state s;
  int err = state_init(&s, n);
  if (err) { state_free(&s); return err; }
  int64_t it = 0;
  for (;;) {
    for (int64_t u = 0; u < n; ++u) s.gf[u] = s.f[s.f[u]];
    memcpy(s.fn, s.f, (size_t)n * sizeof(int32_t));
    for (int64_t e = 0; e < m; ++e) {
      for (int dir = 0; dir < 2; ++dir) {
        int32_t u = pairs[2 * e + dir], v = pairs[2 * e + 1 - dir];
        int32_t hv = s.gf[v], fu = s.f[u];
        if (hv < s.fn[fu]) s.fn[fu] = hv;
        if (hv < s.fn[u]) s.fn[u] = hv;
      }
    }
    for (int64_t u = 0; u < n; ++u) if (s.gf[u] < s.fn[u]) s.fn[u] = s.gf[u];
    int stop = finish_iteration(&s, it, cap, gf_changed, f_changed, snapshots, &err);
    ++it;
    if (err) break;
    if (stop) break;
  }
  if (!err) err = finish_labels(&s, labels);
  if (iterations) *iterations = it;
  state_free(&s);
  return err;
}

/* ---- matrix formulation (driver.py:64-120, dense products) -------------- */

int oracle_fastsv_la_csr(int64_t n, const int64_t* offsets, const int32_t* cols,
                         int64_t cap, int32_t* labels, int64_t* iterations,
                         int64_t* gf_changed, int64_t* f_changed, int32_t* snapshots) {
  size_t bytes = (size_t)(n ? n : 1) * sizeof(int32_t);
  int32_t* f = (int32_t*)malloc(bytes);
  int32_t* gf = (int32_t*)malloc(bytes);
  int32_t* dup = (int32_t*)malloc(bytes);
  int32_t* mngf = (int32_t*)malloc(bytes);
  int32_t* idx_snap = (int32_t*)malloc(bytes);
  int32_t* f_before = (int32_t*)malloc(bytes);
  int err = ORC_OK;
  if (!f || !gf || !dup || !mngf || !idx_snap || !f_before) { err = ORC_ERR_NOMEM; goto out; }
  for (int64_t i = 0; i < n; ++i) f[i] = gf[i] = dup[i] = mngf[i] = idx_snap[i] = (int32_t)i;
  int64_t it = 0;
  for (;;) {
    /* mngf <-min A.gf over non-empty rows (kernels.py:32-68) */
    for (int64_t u = 0; u < n; ++u)
      for (int64_t e = offsets[u]; e < offsets[u + 1]; ++e)
        if (gf[cols[e]] < mngf[u]) mngf[u] = gf[cols[e]];
    memcpy(f_before, f, bytes);
    /* assign_min_scatter(f, idx_snap, mngf) (kernels.py:110-118) */
    for (int64_t u = 0; u < n; ++u) if (mngf[u] < f[idx_snap[u]]) f[idx_snap[u]] = mngf[u];
    /* ewise_min(f, mngf); ewise_min(f, gf) (kernels.py:121-127) */
    for (int64_t u = 0; u < n; ++u) if (mngf[u] < f[u]) f[u] = mngf[u];
    for (int64_t u = 0; u < n; ++u) if (gf[u] < f[u]) f[u] = gf[u];
    int64_t fc = 0, gfc = 0;
    for (int64_t u = 0; u < n; ++u) {
      if (f[u] > f_before[u]) err = ORC_ERR_INVARIANT; /* driver.py:99-100 */
      fc += f[u] != f_before[u];
    }
    memcpy(idx_snap, f, bytes);
    for (int64_t u = 0; u < n; ++u) gf[u] = f[f[u]];          /* extract_grandparent */
    for (int64_t u = 0; u < n; ++u) gfc += dup[u] != gf[u];   /* count_diff(dup, gf) */
    if (it < cap) {
      if (gf_changed) gf_changed[it] = gfc;
      if (f_changed) f_changed[it] = fc;
      if (snapshots) memcpy(snapshots + it * n, f, bytes);
    }
    ++it;
    if (err || gfc == 0) break;
    memcpy(dup, gf, bytes);
  }
  if (iterations) *iterations = it;
  if (!err) {
    for (int64_t u = 0; u < n; ++u) if (f[f[u]] != f[u]) { err = ORC_ERR_INVARIANT; break; }
    if (!err && labels) memcpy(labels, f, bytes);
  }
out:
  free(f); free(gf); free(dup); free(mngf); free(idx_snap); free(f_before);
  return err;
}
