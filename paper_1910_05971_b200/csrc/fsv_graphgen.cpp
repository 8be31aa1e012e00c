// Host-side input preparation: synthetic generators (BASELINE.json configs
// 2-5) and the symmetric CSR builder (restates svcc.build_csr,
// /root/reference/pkg/src/svcc/graph.py:55-97). See include/fsv_graphgen.h.
#include "../../include/fsv_graphgen.h"
#include "philox.h"

#include <omp.h>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

static int g_threads = 0;

extern "C" void fsvg_set_threads(int threads) { g_threads = threads > 0 ? threads : 0; }
extern "C" int fsvg_get_threads(void) { return g_threads > 0 ? g_threads : omp_get_max_threads(); }

static inline int nthreads() { return fsvg_get_threads(); }

static inline uint64_t rand64(uint64_t seed, uint32_t stream, uint64_t index) {
  fsv_u32x4 r = fsv_draw4(seed, stream, index, 0);
  return ((uint64_t)r.v[1] << 32) | r.v[0];
}

extern "C" int fsvg_permutation(int64_t n, uint64_t seed, int32_t* perm) {
  if (n < 0 || n > INT32_MAX) return FSVG_ERR_INPUT;
  if (n == 0) return 0;
  #pragma omp parallel for num_threads(nthreads()) schedule(static)
  for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
  // Fisher–Yates from the top; the draw for position i depends only on i.
  for (int64_t i = n - 1; i > 0; --i) {
    unsigned __int128 p = (unsigned __int128)rand64(seed, FSV_STREAM_PERM, (uint64_t)i) *
                          (unsigned __int128)(uint64_t)(i + 1);
    int64_t j = (int64_t)(uint64_t)(p >> 64);
    int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
  return 0;
}

static int apply_perm(int64_t n, int64_t m, uint64_t seed, int32_t* pairs) {
  std::vector<int32_t> perm;
  try { perm.resize((size_t)n); } catch (...) { return FSVG_ERR_NOMEM; }
  int rc = fsvg_permutation(n, seed, perm.data());
  if (rc) return rc;
  const int32_t* P = perm.data();
  #pragma omp parallel for num_threads(nthreads()) schedule(static)
  for (int64_t i = 0; i < 2 * m; ++i) pairs[i] = P[pairs[i]];
  return 0;
}

extern "C" int64_t fsvg_rmat(int scale, int64_t m, double a, double b, double c,
                             uint64_t seed, int permute, int32_t* pairs) {
  if (scale < 1 || scale > 30 || m < 0 || a < 0 || b < 0 || c < 0 || a + b + c > 1.0)
    return FSVG_ERR_INPUT;
  if (!pairs) return m;
  const double two32 = 4294967296.0;
  const uint64_t tA = (uint64_t)llround(a * two32);
  const uint64_t tAB = (uint64_t)llround((a + b) * two32);
  const uint64_t tABC = (uint64_t)llround((a + b + c) * two32);
  const int groups = (scale + 3) / 4;
  #pragma omp parallel for num_threads(nthreads()) schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    uint32_t row = 0, col = 0;
    for (int g = 0; g < groups; ++g) {
      fsv_u32x4 r = fsv_draw4(seed, FSV_STREAM_RMAT, (uint64_t)i, (uint32_t)g);
      for (int w = 0; w < 4; ++w) {
        int level = g * 4 + w;
        if (level >= scale) break;
        uint64_t x = r.v[w];
        uint32_t bit = 1u << (scale - 1 - level);
        if (x < tA) {
        } else if (x < tAB) {
          col |= bit;
        } else if (x < tABC) {
          row |= bit;
        } else {
          row |= bit; col |= bit;
        }
      }
    }
    pairs[2 * i] = (int32_t)row;
    pairs[2 * i + 1] = (int32_t)col;
  }
  if (permute) {
    int rc = apply_perm((int64_t)1 << scale, m, seed, pairs);
    if (rc) return rc;
  }
  return m;
}

// Grid edge enumeration: horizontal edges k in [0, rows*(cols-1)) are
// (r, c)-(r, c+1) with r = k / (cols-1); vertical edges k' in
// [0, (rows-1)*cols) are (r, c)-(r+1, c). Edge e = k (horizontal) or
// H + k' (vertical) is kept iff its draw >= p_drop * 2^32.
extern "C" int64_t fsvg_grid(int64_t rows, int64_t cols, double p_drop, uint64_t seed,
                             int permute, int32_t* pairs) {
  if (rows < 1 || cols < 1 || rows * cols > INT32_MAX || p_drop < 0 || p_drop > 1)
    return FSVG_ERR_INPUT;
  const int64_t H = rows * (cols - 1);
  const int64_t total = H + (rows - 1) * cols;
  const uint64_t thr = (uint64_t)llround(p_drop * 4294967296.0);
  auto kept = [&](int64_t e) -> bool {
    return (uint64_t)fsv_draw4(seed, FSV_STREAM_GRID, (uint64_t)e, 0).v[0] >= thr;
  };
  const int T = nthreads();
  const int64_t chunk = (total + T - 1) / std::max(T, 1);
  std::vector<int64_t> counts((size_t)T + 1, 0);
  #pragma omp parallel num_threads(T)
  {
    int t = omp_get_thread_num();
    int64_t lo = std::min(total, (int64_t)t * chunk), hi = std::min(total, lo + chunk);
    int64_t cnt = 0;
    for (int64_t e = lo; e < hi; ++e) cnt += kept(e);
    counts[(size_t)t + 1] = cnt;
  }
  for (int t = 0; t < T; ++t) counts[(size_t)t + 1] += counts[(size_t)t];
  const int64_t m = counts[(size_t)T];
  if (!pairs) return m;
  #pragma omp parallel num_threads(T)
  {
    int t = omp_get_thread_num();
    int64_t lo = std::min(total, (int64_t)t * chunk), hi = std::min(total, lo + chunk);
    int64_t o = counts[(size_t)t];
    for (int64_t e = lo; e < hi; ++e) {
      if (!kept(e)) continue;
      int64_t u, v;
      if (e < H) {
        int64_t r = e / (cols - 1), c = e % (cols - 1);
        u = r * cols + c; v = u + 1;
      } else {
        int64_t k = e - H;
        u = k; v = k + cols;
      }
      pairs[2 * o] = (int32_t)u;
      pairs[2 * o + 1] = (int32_t)v;
      ++o;
    }
  }
  if (permute) {
    int rc = apply_perm(rows * cols, m, seed, pairs);
    if (rc) return rc;
  }
  return m;
}

extern "C" int64_t fsvg_forest(int64_t trees, int min_size, int max_size, int extra,
                               uint64_t seed, int permute, int32_t* pairs, int64_t* n_out) {
  if (trees < 0 || min_size < 1 || max_size < min_size || extra < 0) return FSVG_ERR_INPUT;
  std::vector<int64_t> base((size_t)trees + 1, 0), ebase((size_t)trees + 1, 0);
  const uint32_t span = (uint32_t)(max_size - min_size + 1);
  for (int64_t t = 0; t < trees; ++t) {
    uint32_t r = fsv_draw4(seed, FSV_STREAM_TREE_SIZE, (uint64_t)t, 0).v[0];
    int64_t s = min_size + (int64_t)fsv_bounded(r, span);
    base[(size_t)t + 1] = base[(size_t)t] + s;
    ebase[(size_t)t + 1] = ebase[(size_t)t] + (s - 1) + extra;
  }
  const int64_t n = base[(size_t)trees];
  const int64_t m = ebase[(size_t)trees];
  if (n > INT32_MAX) return FSVG_ERR_INPUT;
  if (n_out) *n_out = n;
  if (!pairs) return m;
  #pragma omp parallel for num_threads(nthreads()) schedule(dynamic, 1024)
  for (int64_t t = 0; t < trees; ++t) {
    const int64_t b0 = base[(size_t)t], s = base[(size_t)t + 1] - b0;
    int64_t o = ebase[(size_t)t];
    for (int64_t i = 1; i < s; ++i) {
      uint32_t r = fsv_draw4(seed, FSV_STREAM_TREE_PARENT, (uint64_t)(b0 + i), 0).v[0];
      int64_t parent = (int64_t)fsv_bounded(r, (uint32_t)i);
      pairs[2 * o] = (int32_t)(b0 + i);
      pairs[2 * o + 1] = (int32_t)(b0 + parent);
      ++o;
    }
    for (int e = 0; e < extra; ++e) {
      fsv_u32x4 r = fsv_draw4(seed, FSV_STREAM_TREE_EXTRA, (uint64_t)(t * extra + e), 0);
      pairs[2 * o] = (int32_t)(b0 + fsv_bounded(r.v[0], (uint32_t)s));
      pairs[2 * o + 1] = (int32_t)(b0 + fsv_bounded(r.v[1], (uint32_t)s));
      ++o;
    }
  }
  if (permute) {
    int rc = apply_perm(n, m, seed, pairs);
    if (rc) return rc;
  }
  return m;
}

template <typename ID>
static int64_t csr_build(int64_t n, int64_t m, const ID* pairs, int64_t* offsets,
                         int32_t* cols_out, int64_t* bad_edge) {
  if (n < 0 || n > INT32_MAX || m < 0) return FSVG_ERR_INPUT;
  const int T = nthreads();
  // (1) range check; report the first offending pair in input order
  //     (graph.py:71-75 reports pairs[bad.any(axis=1)][0]).
  int64_t first_bad = INT64_MAX;
  #pragma omp parallel for num_threads(T) reduction(min : first_bad) schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    ID u = pairs[2 * i], v = pairs[2 * i + 1];
    if (u < 0 || u >= (ID)n || v < 0 || v >= (ID)n) first_bad = std::min(first_bad, i);
  }
  if (first_bad != INT64_MAX) {
    if (bad_edge) *bad_edge = first_bad;
    return FSVG_ERR_INPUT;
  }
  // (2) degree count of both orientations, self-loops dropped (graph.py:77-78)
  std::vector<std::atomic<int64_t>> deg((size_t)n);
  #pragma omp parallel for num_threads(T) schedule(static)
  for (int64_t i = 0; i < n; ++i) deg[(size_t)i].store(0, std::memory_order_relaxed);
  #pragma omp parallel for num_threads(T) schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    int64_t u = pairs[2 * i], v = pairs[2 * i + 1];
    if (u == v) continue;
    deg[(size_t)u].fetch_add(1, std::memory_order_relaxed);
    deg[(size_t)v].fetch_add(1, std::memory_order_relaxed);
  }
  std::vector<int64_t> pos((size_t)n + 1, 0);
  for (int64_t i = 0; i < n; ++i) pos[(size_t)i + 1] = pos[(size_t)i] + deg[(size_t)i].load();
  const int64_t raw = pos[(size_t)n];
  int32_t* tmp = (int32_t*)malloc((size_t)std::max<int64_t>(raw, 1) * sizeof(int32_t));
  if (!tmp) return FSVG_ERR_NOMEM;
  // (3) scatter into per-row buckets
  #pragma omp parallel for num_threads(T) schedule(static)
  for (int64_t i = 0; i < n; ++i) deg[(size_t)i].store(pos[(size_t)i], std::memory_order_relaxed);
  #pragma omp parallel for num_threads(T) schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    int64_t u = pairs[2 * i], v = pairs[2 * i + 1];
    if (u == v) continue;
    tmp[deg[(size_t)u].fetch_add(1, std::memory_order_relaxed)] = (int32_t)v;
    tmp[deg[(size_t)v].fetch_add(1, std::memory_order_relaxed)] = (int32_t)u;
  }
  // (4) sort + unique each row (graph.py:80-84 via np.unique on u*n+v)
  std::vector<int64_t> ulen((size_t)n + 1, 0);
  #pragma omp parallel for num_threads(T) schedule(dynamic, 256)
  for (int64_t r = 0; r < n; ++r) {
    int32_t* b = tmp + pos[(size_t)r];
    int32_t* e = tmp + pos[(size_t)r + 1];
    std::sort(b, e);
    ulen[(size_t)r + 1] = std::unique(b, e) - b;
  }
  // (5) offsets = cumsum of unique degrees (graph.py:91-93), compact
  offsets[0] = 0;
  for (int64_t r = 0; r < n; ++r) offsets[r + 1] = offsets[r] + ulen[(size_t)r + 1];
  #pragma omp parallel for num_threads(T) schedule(dynamic, 256)
  for (int64_t r = 0; r < n; ++r)
    memcpy(cols_out + offsets[r], tmp + pos[(size_t)r], (size_t)ulen[(size_t)r + 1] * sizeof(int32_t));
  free(tmp);
  return offsets[n];
}

extern "C" int64_t fsvg_csr_build(int64_t n, int64_t m, const int32_t* pairs,
                                  int64_t* offsets, int32_t* cols, int64_t* bad) {
  return csr_build<int32_t>(n, m, pairs, offsets, cols, bad);
}

extern "C" int64_t fsvg_csr_build64(int64_t n, int64_t m, const int64_t* pairs,
                                    int64_t* offsets, int32_t* cols, int64_t* bad) {
  return csr_build<int64_t>(n, m, pairs, offsets, cols, bad);
}

extern "C" uint64_t fsvg_fnv1a64(const void* data, int64_t nbytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ull;
  for (int64_t i = 0; i < nbytes; ++i) { h ^= p[i]; h *= 0x100000001b3ull; }
  return h;
}
