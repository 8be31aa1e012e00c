/*
 * fsv_graphgen.h — host-side (CPU, OpenMP) input preparation for the FastSV
 * hot path: the synthetic generators of BASELINE.json configs 2–5 and the
 * symmetric CSR builder whose output layout the solver consumes.
 *
 * These sit *beside* the drop-in boundary, not on it:
 *   - fsvg_csr_build restates svcc.build_csr
 *     (/root/reference/pkg/src/svcc/graph.py:55-97): range check -> drop
 *     self-loops -> symmetrise -> deduplicate -> rows sorted ascending.
 *     Output uses int64 row offsets and int32 column ids (the reference uses
 *     int64 for both, graph.py:15-17; int32 ids are what the device stores).
 *   - The generators do not exist in the reference (graphio.py
 *     has only small families); their streams are pinned here by a
 *     counter-based Philox-4x32-10 keyed by (seed, stream, index), see
 *     paper_1910_05971_b200/csrc/philox.h, so CPU and GPU consume identical
 *     edges and every run is reproducible.
 *
 * Conventions: edge lists are int32 pairs laid out [u0, v0, u1, v1, ...].
 * Return values >= 0 are counts; negative values are errors (see below).
 */
#ifndef FSV_GRAPHGEN_H
#define FSV_GRAPHGEN_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSVG_ERR_INPUT (-1)    /* bad parameter or out-of-range edge */
#define FSVG_ERR_NOMEM (-2)

/* Thread count used by the OpenMP loops (0 = library default). */
void fsvg_set_threads(int threads);
int fsvg_get_threads(void);

/* Uniformly random permutation of [0, n) (Fisher–Yates over Philox draws,
 * stream FSV_STREAM_PERM). */
int fsvg_permutation(int64_t n, uint64_t seed, int32_t* perm_out);

/* RMAT (Chakrabarti et al.) with quadrant probabilities (a, b, c, 1-a-b-c):
 * m edges over n = 2^scale vertices, one 32-bit draw per level per edge.
 * permute != 0 relabels endpoints through fsvg_permutation(n, seed).
 * Self-loops and duplicates are kept (build_csr drops them). Returns m. */
int64_t fsvg_rmat(int scale, int64_t m, double a, double b, double c,
                  uint64_t seed, int permute, int32_t* pairs_out);

/* rows x cols 4-neighbour grid, each edge independently dropped with
 * probability p_drop. Pass pairs_out = NULL to get the kept-edge count.
 * Vertex (r, c) has id r*cols + c before the optional permutation. */
int64_t fsvg_grid(int64_t rows, int64_t cols, double p_drop, uint64_t seed,
                  int permute, int32_t* pairs_out);

/* Forest of `trees` random recursive trees with sizes uniform in
 * [min_size, max_size]; local vertex i > 0 attaches to a uniform earlier
 * vertex floor(U*i); plus `extra` uniform intra-tree pairs per tree.
 * *n_out receives the vertex count. pairs_out = NULL -> count only. */
int64_t fsvg_forest(int64_t trees, int min_size, int max_size, int extra,
                    uint64_t seed, int permute, int32_t* pairs_out,
                    int64_t* n_out);

/* Symmetric deduplicated self-loop-free CSR, rows sorted (graph.py:55-97).
 * offsets_out: int64[n+1]; cols_out: capacity >= 2*m int32.
 * Returns m_dir (stored directed entries) or FSVG_ERR_INPUT with
 * *bad_edge = index of the first out-of-range pair (graph.py:71-75). */
int64_t fsvg_csr_build(int64_t n, int64_t m, const int32_t* pairs,
                       int64_t* offsets_out, int32_t* cols_out,
                       int64_t* bad_edge);

/* Same from int64 pairs (the reference's ID dtype). */
int64_t fsvg_csr_build64(int64_t n, int64_t m, const int64_t* pairs,
                         int64_t* offsets_out, int32_t* cols_out,
                         int64_t* bad_edge);

/* FNV-1a 64 over a byte buffer: pins generator streams in tests. */
uint64_t fsvg_fnv1a64(const void* data, int64_t nbytes);

#ifdef __cplusplus
}
#endif
#endif
