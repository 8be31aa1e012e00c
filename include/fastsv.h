/*
 * fastsv.h — C ABI of the B200-native FastSV connected-components solver.
 *
 * This is the drop-in boundary for the reference's hot path, the all-flags
 * FastSV loop `svcc.fastsv_la(g, cfg, record_snapshots)`
 * (/root/reference/pkg/src/svcc/driver.py:64-120) and its vertex-level twin
 * `svcc.fastsv(g)` (algorithms.py:152-167). The reference is pure Python, so
 * its "FFI" is the Python call itself; the ctypes binding a maintainer adds is
 * paper_1910_05971_b200/_native.py (shown in INTEGRATION.md). Plain pointers
 * and sizes only; no torch types.
 *
 * Semantics are bit-exact with the reference: the same per-iteration parent
 * vectors (snapshots), the same iteration count, the same gf_changed and
 * f_changed trace fields (algorithms.py:38-45) and labels equal to the
 * minimum vertex id of each component (graph.py:100-125).
 *
 * Status codes mirror the reference error taxonomy (errors.py:4-19):
 *   FSV_OK 0, FSV_ERR_INPUT 1 (InputError), FSV_ERR_CONTRACT 2 (ValueError),
 *   FSV_ERR_INVARIANT 3 (InvariantError), FSV_ERR_RUNTIME 4 (CUDA/NCCL).
 * fsv_last_error() returns the thread-local message of the last failure.
 *
 * Threading: one solve per context at a time; contexts are independent.
 */
#ifndef FASTSV_H
#define FASTSV_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSV_OK 0
#define FSV_ERR_INPUT 1
#define FSV_ERR_CONTRACT 2
#define FSV_ERR_INVARIANT 3
#define FSV_ERR_RUNTIME 4

#define FSV_ABI_VERSION 5

typedef struct fsv_ctx fsv_ctx;

/* Solver knobs. Zero-initialise for defaults. */
typedef struct fsv_config {
  int32_t max_iters;  /* 0 = run to convergence (the reference has no cap) */
  int32_t batch;      /* iterations queued per host convergence check; 0 = auto */
  int32_t profile;    /* 1 = bracket each kernel with CUDA events (fills *_ms) */
  /* product choice per iteration, svcc.choose_kernel (driver.py:51-61):
   * 0 = reference default (auto, threshold 0.1), 1 = dense only,
   * 2 = sparse only, 3 = auto with `sparse_threshold`. A sparse iteration
   * pushes only the vertices whose gf changed (SpMSpV, kernels.py:71-102);
   * results are identical either way, only the trace's kernel/flops differ. */
  int32_t sparse_policy;
  double sparse_threshold;  /* double: the rule must round like Python's 0.1 * n */
  /* 0 = all-flags FastSV on the fast path. FSV_HOOKING_SET | flag bits runs
   * the reference's HookingConfig variant (algorithms.py:28-35,85-114) on the
   * generic variant kernels: FSV_HOOKING_SET alone is simplified_sv
   * (algorithms.py:66-76,145-149, trace-identical to all flags off). The
   * variant trace reports kernel "none" (0) and flops 0, as the reference. */
  int32_t hooking;
  /* multi-rank exchange of the next-parent vector:
   * 0 = dense iterations allreduce-min, sparse iterations exchange only the
   *     entries each rank lowered (allgather of (index, value) lists, bytes
   *     proportional to the delta; host in the loop per iteration);
   * 1 = allreduce-min every iteration (the loop may run as one CUDA graph
   *     with the collective captured). Results are identical. */
  int32_t exchange;
} fsv_config;

#define FSV_HOOKING_SET 0x100
#define FSV_HOOK_GRANDPARENT 1        /* hook gf[v] rather than f[v] */
#define FSV_HOOK_STOCHASTIC 2         /* f[f[u]] <-min, one commit per iteration */
#define FSV_HOOK_AGGRESSIVE 4         /* f[u] <-min */
#define FSV_HOOK_EARLY_TERMINATION 8  /* stop on gf stability (only with all four) */

/* Result summary of the last solve. */
typedef struct fsv_stats {
  int32_t iterations;       /* == reference RunResult.iterations */
  int32_t component_count;  /* == Labeling.component_count */
  int64_t n;
  int64_t m_dir;            /* stored directed entries of the uploaded CSR */
  int64_t oriented_entries; /* entries the device layout stores (one per edge) */
  int32_t hub_slots;        /* hub table size actually used */
  int32_t host_syncs;       /* convergence-flag reads the host made */
  int32_t kernel_launches;  /* kernels launched by the solve */
  float solve_ms;           /* device time, first kernel to convergence flag */
  /* profile = 1 only: summed device time of the kernels of the iterations
   * that ran (speculative launches past convergence excluded) */
  float hook_ms, hubfix_ms, shortcut_ms, first_ms, allreduce_ms, push_ms;
  int32_t hook_launches;
  int32_t sparse_iterations;  /* iterations that ran the sparse push */
  /* multi-rank: exchanges by kind and bytes this rank sent (allreduce: ring
   * bus bytes 2(P-1)/P*4n; delta: 8 bytes per pair to each other rank) */
  int32_t dense_exchanges, delta_exchanges;
  int64_t exchange_bytes;
  int32_t minority_iterations;  /* dense iterations that ran the minority sweep instead of the full sweep */
  int32_t reserved;
} fsv_stats;

const char* fsv_last_error(void);
int fsv_abi_version(void);
int fsv_device_count(int* count);

/* Context bound to one CUDA device; creates its own non-blocking stream. */
int fsv_create(int device, fsv_ctx** out);
int fsv_destroy(fsv_ctx* ctx);

/* Hub table size used by the NEXT upload: <0 = no hubs, 0 = auto
 * (top-degree vertices up to 47104 shared-memory slots: 192 KB with the hot
 * accumulators, which keeps enough L1 for the global gathers), >0 = at most
 * that, up to 55296. */
int fsv_set_hub_slots(fsv_ctx* ctx, int slots);

/* Column-range tiling of the NEXT upload's layout, for graphs without a
 * hub table and without rows over 512 entries whose vertex vectors overflow
 * L2 (BASELINE configs 3 and 4): every row is split into per-tile segments
 * and the layout holds tile 0's segments, then tile 1's, ..., so the dense
 * sweep gathers from (and reduces into) one L2-resident slice of the vertex
 * vectors at a time. Results are identical; the layout build costs one
 * count + compact pass per tile. 0 = off (default), > 0 = vertices per
 * tile, < 0 = auto (8 M vertices = 32 MB slices). */
int fsv_set_tile_width(fsv_ctx* ctx, int64_t vertices);

/* Minority sweep (default on). In a dense iteration from the third on, of a
 * hub-table layout held by one rank: when the vertices whose grandparent
 * differs from that of the most connected vertex have a small degree sum
 * (at most 1/16 of the stored directed entries), only the edges incident to
 * them are visited (a push in both directions along their CSR rows) instead
 * of sweeping every stored entry; an entry whose endpoints carry the same
 * grandparent contributes nothing. Results are identical; 0 turns it off. */
int fsv_set_minority_sweep(fsv_ctx* ctx, int enable);

/* Use an external stream (e.g. torch.cuda.current_stream().cuda_stream);
 * 0 restores the context's own stream. */
int fsv_set_stream(fsv_ctx* ctx, void* cuda_stream);

/*
 * Upload a symmetric CSR (the reference CsrGraph layout, graph.py:20-52:
 * rows sorted, deduplicated, self-loop free) and build the device layout.
 *   row_offsets: n+1 entries of the FULL graph (int64, as the reference)
 *   col_indices: the entries of rows [row_begin, row_end), i.e. the slice
 *                [row_offsets[row_begin], row_offsets[row_end]); int32 ids
 * Single GPU: row_begin = 0, row_end = n. With an attached NCCL communicator
 * every rank passes its own disjoint row range (1D partition).
 * Host buffers may be pageable or pinned. Replaces svcc.build_csr's product
 * being handed to fastsv_la (driver.py:64).
 */
int fsv_upload_csr(fsv_ctx* ctx, int64_t n, const int64_t* row_offsets,
                   const int32_t* col_indices, int64_t row_begin, int64_t row_end);

/*
 * Same from DEVICE memory (a CsrGraph already resident in HBM, e.g. torch
 * tensors): d_row_offsets holds the n+1 int64 offsets of the full graph,
 * d_col_indices the int32 columns of rows [row_begin, row_end) (the slice
 * starting at row_offsets[row_begin]). Both arrays are BORROWED: the context
 * reads them in place (sparse iterations and f_1 read the symmetric CSR) and
 * they must stay valid and unchanged until the next upload or fsv_destroy.
 * Only the layout is built; nothing is copied.
 */
int fsv_upload_csr_device(fsv_ctx* ctx, int64_t n, const int64_t* d_row_offsets,
                          const int32_t* d_col_indices, int64_t row_begin, int64_t row_end);

/* Same with int64 column ids (the reference's ID_DTYPE, graph.py:15-17). */
int fsv_upload_csr64(fsv_ctx* ctx, int64_t n, const int64_t* row_offsets,
                     const int64_t* col_indices, int64_t row_begin, int64_t row_end);

/*
 * Upload a raw edge list and build the CsrGraph on the device with
 * svcc.build_csr's semantics (graph.py:55-97): every pair range-checked
 * (status 1, "edge (u, v) out of range for n=N" for the first offending pair
 * in input order, graph.py:71-75), self-loops dropped, both orientations
 * stored, duplicates merged, rows sorted. Then the device layout is built as
 * by fsv_upload_csr for rows [row_begin, row_end). pairs: m (u, v) pairs,
 * 2*m ids, int32 or int64 (the reference's ID_DTYPE).
 */
int fsv_upload_edges(fsv_ctx* ctx, int64_t n, int64_t m, const int32_t* pairs,
                     int64_t row_begin, int64_t row_end);
int fsv_upload_edges64(fsv_ctx* ctx, int64_t n, int64_t m, const int64_t* pairs,
                       int64_t row_begin, int64_t row_end);

/*
 * Copy the resident symmetric CSR to host: row_offsets (n+1, int64, full
 * graph) and the columns of this context's rows (csr_entries of them; the
 * count is returned in *csr_entries when cols is NULL). Lets callers obtain
 * the CsrGraph that fsv_upload_edges built (CsrGraph.row_offsets /
 * col_indices, graph.py:20-52).
 */
int fsv_get_csr(fsv_ctx* ctx, int64_t* row_offsets, int32_t* cols, int64_t* csr_entries);

/* Run FastSV to convergence on the resident graph. Labels stay on device. */
int fsv_solve(fsv_ctx* ctx, const fsv_config* cfg, fsv_stats* stats);

/* The fsv_stats of the last solve (as fsv_solve fills them). */
int fsv_get_stats(fsv_ctx* ctx, fsv_stats* stats);

/* Copy results of the last solve to host buffers.
 *   labels: n int32 (or int64 via fsv_get_labels64)
 *   trace:  cap entries each of gf_changed / f_changed (int64) and
 *           per-iteration device milliseconds (float); any may be NULL. */
int fsv_get_labels(fsv_ctx* ctx, int32_t* labels);
int fsv_get_labels64(fsv_ctx* ctx, int64_t* labels);
int fsv_get_trace(fsv_ctx* ctx, int64_t* gf_changed, int64_t* f_changed,
                  float* elapsed_ms, int32_t cap);
/* Same plus the product kind per iteration (0 dense, 1 sparse) and its
 * flops (dense: m_dir; sparse: degree sum of the pushed vertices), the
 * IterationTrace.kernel / .flops fields (algorithms.py:38-45). */
int fsv_get_trace_ex(fsv_ctx* ctx, int64_t* gf_changed, int64_t* f_changed,
                     float* elapsed_ms, int32_t* kernel, int64_t* flops, int32_t cap);

/* The Labeling of the last solve, computed on the device (the reference's
 * labeling_from_parents, graph.py:109-125; the star check already ran in
 * the final vertex pass and failed the solve with FSV_ERR_INVARIANT):
 *   labels: n int64 (the reference's ID_DTYPE), or NULL
 *   reps, sizes: the component representatives in ascending order (the
 *           minimum id of each component) and their vertex counts, `cap`
 *           entries each, or NULL
 *   count:  receives the component count (Labeling.component_count).
 * Call with reps = sizes = NULL first to size the buffers. */
int fsv_get_labeling(fsv_ctx* ctx, int64_t* labels, int64_t* reps, int64_t* sizes, int64_t cap,
                     int64_t* count);

/* One call: solve + labels + iteration count + trace (the fastsv_la shape). */
int fsv_run(fsv_ctx* ctx, const fsv_config* cfg, int32_t* labels,
            int32_t* iterations, int64_t* gf_changed, int64_t* f_changed,
            int32_t trace_cap);

/* Solve while copying every committed parent vector f_k (k = 1..I) into
 * snapshots[(k-1)*n .. k*n) (record_snapshots=True, driver.py:109-112).
 * Fails with FSV_ERR_CONTRACT if more than snap_cap iterations run. */
int fsv_run_snapshots(fsv_ctx* ctx, const fsv_config* cfg, int32_t* labels,
                      int32_t* iterations, int64_t* gf_changed, int64_t* f_changed,
                      int32_t* snapshots, int32_t snap_cap);

/* ---- multi-GPU (one process per GPU, 1D edge partition) ---- */

/* Fills 128 bytes with an ncclUniqueId (rank 0), to be broadcast by the host. */
int fsv_nccl_unique_id(void* id128);
/* Attach a communicator; per iteration the next-parent vector is merged with
 * ncclAllReduce(ncclInt32, ncclMin) after the hooking phase. */
int fsv_nccl_attach(fsv_ctx* ctx, const void* id128, int nranks, int rank);

/* ---- emulated rank group (one device; tests of the partitioned path) ----
 * `count` (1..8) contexts on ONE device, each uploaded with a disjoint row
 * range of the same graph (together covering [0, n): the 1D partition of the
 * multi-GPU path), solved in lockstep on rank 0's stream: every rank's
 * hooking kernels, then one kernel that min-merges the ranks' next-parent
 * vectors (what ncclAllReduce(ncclInt32, ncclMin) does across processes,
 * SURVEY §8a E4), then every rank's vertex pass. f_1 is assembled the same
 * way. Runs the rank-partitioned kernels (row-filtered push, per-rank hub
 * fix-up, f_1 assembly, host-batched loop) with fewer GPUs than ranks; no
 * kernel waits on another. Results are replicated: each context's labels
 * and trace equal the single-context solve; stats/snapshots are rank 0's
 * (trace flops are the group's sum). */
int fsv_group_solve(fsv_ctx* const* ctxs, int count, const fsv_config* cfg, fsv_stats* stats);
int fsv_group_run_snapshots(fsv_ctx* const* ctxs, int count, const fsv_config* cfg, int32_t* labels,
                            int32_t* iterations, int64_t* gf_changed, int64_t* f_changed,
                            int32_t* snapshots, int32_t snap_cap);

#ifdef __cplusplus
}
#endif
#endif
