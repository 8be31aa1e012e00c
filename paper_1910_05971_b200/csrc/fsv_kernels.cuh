// FastSV device kernels for sm_100a (B200). Integer, HBM/L2-bound, no tensor
// cores: nothing on this path is a dense contraction.
//
// One FastSV iteration k (all flags; algorithms.py:79-91 == driver.py:81-117)
// maps onto two launches over buffers F = f_k, G = gf_k, N = f_{k+1}
// (pre-initialised to gf_k, which folds the shortcut f <-min gf, E1):
//
//   k_hook      edge-parallel over the oriented layout (each undirected edge
//               stored once, in the row of its lower-(degree,id) endpoint):
//               row side   mngf run-min -> N[u]   (aggressive hook)
//               column side gf[u]       -> N[v]   (same rule, v <- u)
//               gf of the top-H degree vertices ("hubs") is read from shared
//               memory; column-side writes aimed at hubs are min-reduced into
//               a compact hub accumulator instead of random N atomics, which
//               the same launch applies after a grid barrier (hub fix-up;
//               k_hubfix when built with FSV_FUSE_HUBFIX=0). A sparse
//               iteration takes the push branch of the same kernel (both
//               hooks per contribution), and a late dense iteration the
//               minority sweep (hook_minority) when few vertices are left
//               outside the majority grandparent.
//   k_shortcut  vertex-parallel: after a dense sweep the deferred stochastic
//               hooks N[F[u]] <-min N[u] of the lowered vertices, then
//               gf_{k+1} = N[N], change counters, star and monotonicity
//               checks, next N init, hub gf refresh, and the device-side
//               convergence flag (last-block ticket).
//
// Iteration 1 is closed-form (F = G = id): f_1[u] = min(u, min neighbour id),
// computed by every solve from the sorted CSR rows (k_f1_solve), so k_first
// does iteration 1 including its shortcut phase in one vertex-parallel pass.
//
// Writes into N are min-atomics filtered by the read-only gf_k: N[x] <= gf_k[x]
// always and gf_k[F[x]] <= gf_k[x], so val >= gf_k[x] makes both hooks
// no-ops.
//
// Stochastic hooks of a dense iteration are deferred to the vertex pass: the
// dense sweep only applies the aggressive hooks (N[x] <-min val), which leaves
// N[u] = min(gf_k[u], mngf[u]); k_shortcut then applies f[f_k[u]] <-min
// mngf[u] once per lowered vertex (N[u] < gf_k[u] implies N[u] = mngf[u];
// for the others mngf[u] >= gf_k[u] >= gf_k[f_k[u]] >= N[f_k[u]] is a no-op)
// from coalesced streams, instead of a parent gather and a second reduction
// per contributing entry inside the sweep. A sparse (push) iteration applies
// both hooks inline.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace fsv {

#ifdef FSV_DEBUG_TIMING
// dev-only phase timestamps of the sparse path: [block][0..3]
__device__ unsigned long long g_dbg_t[1024 * 4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define DBG_T(slot) do { if (threadIdx.x == 0) g_dbg_t[blockIdx.x * 4 + (slot)] = gtimer(); } while (0)
#else
#define DBG_T(slot) do { } while (0)
#endif

constexpr int INF = 0x7fffffff;
// Oriented layout entry codes (uint32):
//   header  HDR | u          first entry of the row of vertex u
//   edge    [HUB] | v/slot   neighbour v (or its hub slot) of the current row
constexpr uint32_t HDR = 0x80000000u;
constexpr uint32_t HUB = 0x40000000u;    // edge column is a hub: low bits = slot
constexpr uint32_t IDMASK = 0x3fffffffu;
#ifndef FSV_HOOK_THREADS
#define FSV_HOOK_THREADS 1024
#endif
#ifndef FSV_STEPS
#define FSV_STEPS 4
#endif
constexpr int EPL = 8;                   // contiguous entries per lane per step
constexpr int STEP = 32 * EPL;           // entries per warp step
constexpr int STEPS = FSV_STEPS;         // steps per span
constexpr int SPAN = STEP * STEPS;       // entries per warp task
constexpr int HOOK_THREADS = FSV_HOOK_THREADS;
constexpr int PUSH_SCRATCH_BYTES = HOOK_THREADS * 40;  // s_start, s_excl (8 B), s_val, s_src (4 B), s_list (16 B)
// Column-side minima aimed at the HOT_ACC most connected hubs are combined in
// shared memory per CTA and flushed once at the end: a top hub can be the
// target of ~1e5 reductions per iteration, which would otherwise serialise
// on the one L2 slice that owns its line.
#ifndef FSV_HOT_ACC
#define FSV_HOT_ACC 2048
#endif
constexpr int HOT_ACC = FSV_HOT_ACC;
// Steps in which no lane has more than FSV_REC entries that differ from their
// row's gf take the record path of k_hook (per-entry emissions, no scan);
// 0 disables it. At most 2 records are held in registers.
#ifndef FSV_REC
#define FSV_REC 2
#endif
static_assert(FSV_REC >= 0 && FSV_REC <= 2, "FSV_REC must be 0, 1 or 2");
constexpr int SMEM_OPTIN_INTS = 232448 / 4;   // 227 KB opt-in dynamic shared memory per CTA
constexpr int SC_THREADS = 512;
constexpr int NCOUNT = 16;               // counter slots per iteration
enum { C_GF = 0, C_F = 1, C_NONSTAR = 2, C_ROOTS = 3, C_VIOL = 4,   // vertex-pass counters
       C_FLOPS = 5, C_CHUNKS = 6, C_BARRIER = 8,       // push bookkeeping
       C_FIXBAR = 9,                                   // hub fix-up barrier of the dense hook
       C_SPANS = 10,                                   // dynamic task counter of the dense hook
       C_SCBAR = 11, C_SCBAR2 = 12,                    // grid barriers of the vertex pass (deferred hooks)
       C_MDEG = 13, C_MBAR = 14,                       // minority sweep: degree sum of the listed vertices, barrier,
       C_MDONE = 15 };                                 // 1 when it replaced this iteration's dense sweep (stats)

// ---- memory helpers -------------------------------------------------------

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Streamed once per iteration: evict first from L2 so the parent vectors
// stay L2-resident. L1 may allocate: a lane's two 16-byte halves share sectors.
// A lane's 8 entries of a step as one 256-bit load (sm_100): one request per
// sector, and no L1 allocation (FSV_STREAM_NA) so the ~60 KB of L1 next to
// the hub table stay with the gathers.
#ifndef FSV_STREAM_V8
#define FSV_STREAM_V8 1
#endif
#ifndef FSV_STREAM_NA
#define FSV_STREAM_NA 1
#endif
struct Entries8 {
  uint32_t c[8];
};
__device__ __forceinline__ Entries8 ld_stream8(const uint4* p, uint64_t pol) {
  Entries8 r;
#if FSV_STREAM_V8
#if FSV_STREAM_NA
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
#else
  asm volatile("ld.global.nc.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
#endif
               : "=r"(r.c[0]), "=r"(r.c[1]), "=r"(r.c[2]), "=r"(r.c[3]), "=r"(r.c[4]), "=r"(r.c[5]),
                 "=r"(r.c[6]), "=r"(r.c[7]) : "l"(p), "l"(pol));
#else
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.c[0]), "=r"(r.c[1]), "=r"(r.c[2]), "=r"(r.c[3]) : "l"(p), "l"(pol));
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.c[4]), "=r"(r.c[5]), "=r"(r.c[6]), "=r"(r.c[7]) : "l"(p + 1), "l"(pol));
#endif
  return r;
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}

#ifdef FSV_CHECKS
// Checked build (tests only, -DFSV_CHECKS): every read-only vertex-array load
// and every min-reduction of the FastSV solve kernels must hit one of the
// buffers the host registered for this solve, else the kernel traps. Ranges
// are empty (checks off) outside fastsv solves.
constexpr int kChkRed = 32, kChkLd = 96;   // room for an emulated rank group of 8 contexts
struct ChkRanges {
  const int* rlo[kChkRed];
  const int* rhi[kChkRed];
  int nr;
  const int* lo[kChkLd];
  const int* hi[kChkLd];
  int nl;
};
__device__ ChkRanges g_chk;
__device__ __noinline__ void chk_fail(const void* p, int red) {
  printf("FSV_CHECKS: %s outside the registered buffers: %p (block %d thread %d)\n",
         red ? "reduction" : "load", p, blockIdx.x, threadIdx.x);
  __trap();
}
__device__ __forceinline__ void chk_red(const int* p) {
  const int nr = g_chk.nr;
  if (!nr) return;
  for (int i = 0; i < nr; ++i)
    if (p >= g_chk.rlo[i] && p < g_chk.rhi[i]) return;
  chk_fail(p, 1);
}
__device__ __forceinline__ void chk_ld(const int* p) {
  const int nl = g_chk.nl;
  if (!nl) return;
  for (int i = 0; i < nl; ++i)
    if (p >= g_chk.lo[i] && p < g_chk.hi[i]) return;
  chk_fail(p, 0);
}
#define FSV_CHK_RED(p) chk_red(p)
#define FSV_CHK_LD(p) chk_ld(p)
#else
#define FSV_CHK_RED(p) do { } while (0)
#define FSV_CHK_LD(p) do { } while (0)
#endif

__device__ __forceinline__ int ldg(const int* p) {
  FSV_CHK_LD(p);
  return __ldg(p);
}

__device__ __forceinline__ void red_min(int* p, int v) {
  FSV_CHK_RED(p);
  asm volatile("red.relaxed.gpu.global.min.s32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void red_min_shared(uint32_t saddr, int v) {
  asm volatile("red.shared.min.s32 [%0], %1;" :: "r"(saddr), "r"(v) : "memory");
}

// Hub accumulator slot -> int index. FSV_ACC_STRIDE > 1 spreads the first
// ACC_SPREAD slots (the shared-memory hubs, whose accumulators take most of
// the column-side reductions) one per STRIDE ints; tier slots beyond stay
// packed.
// Default 2: with packed slots (1) eight accumulators share a 32-byte sector,
// the reductions aimed at them queue at the L2 slice that owns it, and the
// dense hook's time depended on where the array sat in its 2 MB page (config
// 2: 0.501-0.524 ms over FSV_HPAD/FSV_VPAD shifts); one slot per 8 bytes
// gives 0.508-0.512 ms at every placement (4 and 8 the same, 32 slower).
#ifndef FSV_ACC_STRIDE
#define FSV_ACC_STRIDE 2
#endif
constexpr int ACC_SPREAD = 65536;
__host__ __device__ __forceinline__ long long acc_at(long long s) {
  return FSV_ACC_STRIDE == 1 ? s
         : (s < ACC_SPREAD ? s * FSV_ACC_STRIDE : (long long)ACC_SPREAD * FSV_ACC_STRIDE + (s - ACC_SPREAD));
}
// Shared-memory hub slots (< H <= ACC_SPREAD) never reach the packed tail, so
// the kernels without the rank tier index with one multiply.
template <bool TIER>
__device__ __forceinline__ long long acc_idx(int s) {
  return TIER ? acc_at(s) : (long long)s * FSV_ACC_STRIDE;
}
__host__ __device__ __forceinline__ long long acc_len(long long slots) {
  return slots <= 0 ? 0 : acc_at(slots - 1) + 1;
}

// ---- argument blocks --------------------------------------------------------

// Report of a graph-mode solve, packed on the device by the last block of
// the final iteration (trace of the first STAGE_ITERS iterations, done flag)
// so the host fetches it with one copy.
constexpr int STAGE_ITERS = 64;
static_assert(NCOUNT == 16, "SolveReport holds 16 counters per iteration");
struct SolveReport {
  int done;                                        // iteration (>0 converged, <0 cap reached)
  int iters;                                       // iterations staged below (0: more than STAGE_ITERS)
  unsigned long long cnt[STAGE_ITERS * 16];        // NCOUNT counters per iteration
  int mode[STAGE_ITERS + 2];
  unsigned long long ts[STAGE_ITERS + 2];
};

// Device-side loop control. Graph mode runs the iteration loop inside a
// CUDA-graph conditional WHILE node: kernels read the iteration number from
// *iterp, the vertex pass's last block advances it and sets the condition.
struct LoopCtl {
  int* iterp;                        // graph mode: current iteration (>= 2)
  unsigned long long* cnt_base;      // counters of iteration 1 (NCOUNT per iteration)
  unsigned long long* tstamp;        // per-iteration end time (%globaltimer, ns)
  unsigned long long cond;           // cudaGraphConditionalHandle of the WHILE loop
  unsigned long long cond_next;      // IF handle guarding the body's next iteration (0: none)
  SolveReport* rep;                  // graph mode: the solve's report (device memory) or null
  int* mode_base;                    // mode[] of the whole solve (for the report)
  int graph;                         // 0 host loop, 1 inside the graph, 2 k_first before it
  int* X;                            // graph mode: the two rotating parent buffers; iteration k
  int* Y;                            // reads F = f_{k-1} and writes N = f_k by its parity
};

// Graph mode: the loop body is one iteration, so the buffers rotate by the
// iteration number read on the device (k_first leaves f_1 in Y).
__device__ __forceinline__ void loop_bufs(const LoopCtl& lc, int it, int*& F, int*& N) {
  F = (it & 1) ? lc.X : lc.Y;
  N = (it & 1) ? lc.Y : lc.X;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int loop_iter(const LoopCtl& lc, int iter) {
  return lc.graph == 1 ? __ldcg(lc.iterp) : iter;   // written by the previous kernel
}

// Early exit after convergence: in graph mode the loop condition must drop.
__device__ __forceinline__ bool converged_exit(const int* done, const LoopCtl& lc) {
  if (__ldcg(done)) {
    if (lc.graph == 1 && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(lc.cond, 0u);
    return true;
  }
  return false;
}

// Sparse iteration (push). Phase A: one warp per delta region takes the
// changed vertices 32 at a time; rows of at most PUSH_BIG entries are pushed
// by that warp right away (the batch's rows flattened, 8 entries per lane per
// pass), longer rows are cut into PUSH_CHUNK-entry chunks appended to a
// global list. Phase B (after a grid barrier) pushes the chunks, one warp per
// chunk, so a high-degree vertex is spread over the whole GPU.
struct PushChunk {
  long long pos_cnt; // first column index of the chunk (rank-local, < 2^48) | entries in the chunk << 48
  int val;           // gf[v] pushed to every neighbour
  int src;           // v itself (the minority sweep pulls the neighbours' gf back into N[v])
};

struct PushArgs {
  const int* list;        // delta regions of the previous vertex pass
  const int* count;
  long long rcap;
  int nregions;
  const int64_t* off;     // full symmetric CSR offsets (n+1)
  const int* cols;        // columns of rows [row_begin, row_end)
  long long col_base;     // off[row_begin]
  int row_begin, row_end;
  const int* F;
  const int* G;
  int* N;
  const int* mode;        // mode[iter]
  int iter;
  unsigned long long* flops;    // this iteration's pushed-entry count
  unsigned long long* nchunks;  // long-row chunk list length
  PushChunk* chunks;            // long-row chunks
  unsigned* barrier;            // grid barrier counter of this iteration
};

struct HookArgs {
  const uint32_t* ecol;   // oriented entries (headers + edges), padded to SPAN
  long long nspans;       // warp tasks of NSTEP consecutive STEP-entry steps
  const int* span_row;    // vertex of the row open at each task start, -1 if none
  const int* F;           // f_k
  const int* G;           // gf_k
  int* N;                 // f_{k+1}, pre-initialised to gf_k
  const int* G_hub;       // gf_k of all tier slots, degree-rank order (compact)
  int H;                  // shared-memory slots (multiple of 4)
  int HT;                 // all tier slots: [0,H) shared memory, [H,HT) the L2 rank tier
  int* hub_acc;           // column-side minima aimed at tier slots
  const int* hub_id;      // slot -> vertex (fused hub fix-up)
  unsigned* fix_barrier;  // grid barrier before the fused hub fix-up
  unsigned* task_ctr;     // dynamic tail of the dense task loop (FSV_DYN_TAIL)
  const int* done;        // convergence flag (iteration number, 0 = running)
  const int* mode;        // mode[iter]: 0 dense pull (this layout), 1 sparse push
  int iter;
  PushArgs push;
  LoopCtl lc;
  // minority sweep (hub-table layouts): see hook_minority
  long long n;            // vertices
  int* mlist;             // the vertex pass's delta regions, free during a dense hook
  int* mcount;
  const int* off32;       // int32 copy of the CSR offsets when they fit, else null
  long long minority_thr; // degree sum up to which the minority sweep replaces the dense sweep (< 0: off)
};

// Changed-gf ("delta") list written by the vertex pass: warp w owns
// list[w*rcap, w*rcap + count[w]) so no global atomics are needed.
// policy: 0 auto (sparse iff gf_changed < threshold*n, driver.py:51-61),
// 1 dense only, 2 sparse only. mode[k] (k = 1-based iteration) is written by
// the last block of iteration k-1: 0 dense product, 1 sparse push.
struct DeltaOut {
  int* list;
  int* count;
  long long rcap;
  int* mode;
  int policy;
  double threshold;
  long long n_total;      // global vertex count for the threshold rule
};

struct ShortcutArgs {
  int* F;                 // in: f_k; out: gf_{k+1} (next N init)
  int* G;                 // in: gf_k; out: gf_{k+1}
  int* N;                 // f_{k+1} (the stochastic hooks of a dense iteration are applied to it here)
  const int* mode;        // mode[iter]: 0 after a dense sweep (aggressive hooks only), 1 after a push
  long long n;
  const int* hub_id;
  int* G_hub;
  int H;                  // tier slots refreshed here (all of them)
  unsigned long long* cnt;  // this iteration's NCOUNT counters
  unsigned* partials;       // per-block partial counters [grid][8]
  unsigned int* ticket;
  int* done;
  int iter;               // 1-based iteration number
  int max_iter;           // stop flag raised when reached without converging
  DeltaOut dl;            // changed-gf list for a following sparse iteration
  LoopCtl lc;
};

// ---- emission of one hook contribution -------------------------------------

// Aggressive hook of the dense sweep: value `val` (a row's run minimum, or a
// row's gf on the column side) aimed at vertex u whose gf is gu. The
// stochastic hook is deferred to the vertex pass (k_shortcut).
__device__ __forceinline__ void emit_agg(int u, int gu, int val, int* __restrict__ N) {
  if (val < gu) red_min(N + u, val);
}

// k_hook applies the hub accumulator itself after a grid barrier instead of
// a separate k_hubfix launch.
#ifndef FSV_FUSE_HUBFIX
#define FSV_FUSE_HUBFIX 1
#endif
// A scan step with emissions on at least FSV_DENSE_LANES lanes puts the warp
// in dense mode: its next step goes straight to the scan path (no
// differing-entry count). 0 disables; used by the hub-table kernels (skewed
// graphs, where the dense iterations have most entries differing).
// Dense task loop: the last FSV_DYN_TAIL rounds of tasks are handed out by
// an atomic counter (0: fully static round-robin).
// Changed-vertex lists of the vertex passes hold 4-vertex groups with a
// change mask (one ballot per group); the push expands them.
#ifndef FSV_DELTA_GROUPS
#define FSV_DELTA_GROUPS 1
#endif
#ifndef FSV_DYN_TAIL
#define FSV_DYN_TAIL 2
#endif
#ifndef FSV_DYN_NOHUB
#define FSV_DYN_NOHUB 0
#endif
#ifndef FSV_DENSE_LANES
#define FSV_DENSE_LANES 16
#endif
// Dev speed-of-light probes (wrong results, timing only): bit 0 drops the
// dense hook's emissions, bit 1 its global gathers.
#ifndef FSV_SOL
#define FSV_SOL 0
#endif
// One gathered gf value per entry: hub edges from the shared-memory table
// (32-bit shared address, no generic conversion), everything else from
// global through the read-only path. Both loads are predicated, no branch.
__device__ __forceinline__ int gather_gf(uint32_t c, uint32_t s_base, const int* __restrict__ G) {
#ifdef FSV_CHECKS
  if (!(c & HUB)) chk_ld(G + (c & IDMASK));
#endif
  int v;
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "@p  ld.shared.b32 %0, [%2];\n\t"
      "@!p ld.global.nc.b32 %0, [%3];\n\t}"
      : "=r"(v)
      : "r"(c & HUB), "r"(s_base + (c << 2)), "l"(G + (c & IDMASK)));
  return v;
}

// ---- sparse iteration: push over the changed-gf list --------------------------
// Iteration k >= 2 only needs the directed entries (u -> v) with gf[v]
// changed in iteration k-1: every other contribution is dominated by the
// previous iteration's aggressive hook (f_{k-1}[u] <= min_{v in N(u)} gf_{k-2}[v],
// and gf[F[u]] <= f_{k-1}[u]). So v pushes gf[v] to each neighbour u of the
// symmetric CSR: N[u] <-min, N[F[u]] <-min, with the usual filters. This is
// the reference's SpMSpV (kernels.py:71-102) without the mngf accumulator.


constexpr int PUSH_CHUNK = 256;  // entries per phase-A pass (8 per lane)
#ifndef FSV_PUSH_BIG
#define FSV_PUSH_BIG 128
#endif
#ifndef FSV_PUSH_BCHUNK
#define FSV_PUSH_BCHUNK 64
#endif
constexpr int PUSH_BIG = FSV_PUSH_BIG;        // rows longer than this go to the chunk list
constexpr int PUSH_BCHUNK = FSV_PUSH_BCHUNK;  // entries per long-row chunk (phase B)
static_assert(PUSH_BCHUNK % 32 == 0 && PUSH_BIG <= 8192, "push chunk shapes");

// Push val[j] to neighbour u[j] (u < 0: no entry): N[u] <-min val when it
// can lower gf[u] (aggressive), then N[F[u]] <-min val when it can lower
// gf[F[u]] (stochastic). The second filter matters here: every neighbour of
// a pushed vertex receives the same value, and their parents are often one
// root, so unfiltered reductions would pile onto one address. All loads of
// the lane are issued together.
// BIDIR (minority sweep of a dense iteration): the neighbour's gf is also
// pulled back into the source vertex, N[src] <-min gf[u], and only the
// aggressive hooks are applied (the vertex pass defers the stochastic ones).
// ONE_SRC: the whole warp pushes one vertex's entries (a long-row chunk), so
// the pull-back is one warp-reduced minimum: a straggler of degree 25,000
// whose neighbours all carry the majority value would otherwise queue 25,000
// reductions on the one address N[src].
template <int PER, bool BIDIR, bool ONE_SRC = false>
__device__ __forceinline__ void push_entries(const int (&u)[PER], const int (&val)[PER], const int (&src)[PER],
                                             const int* __restrict__ F, const int* __restrict__ G,
                                             int* __restrict__ N) {
  int gt[PER], t[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) gt[j] = u[j] >= 0 ? ldg(G + u[j]) : INF;
  if (BIDIR) {
    int back = INF;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (u[j] >= 0 && val[j] < gt[j]) red_min(N + u[j], val[j]);
      if (ONE_SRC) back = min(back, gt[j]);
      else if (u[j] >= 0 && gt[j] < val[j]) red_min(N + src[j], gt[j]);
    }
    if (ONE_SRC) {
      back = __reduce_min_sync(0xffffffffu, back);
      if ((threadIdx.x & 31) == 0 && back < val[0]) red_min(N + src[0], back);
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    t[j] = -1;
    if (u[j] >= 0 && val[j] < gt[j]) {
      red_min(N + u[j], val[j]);
      t[j] = ldg(F + u[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    if (t[j] == u[j]) t[j] = -1;
    gt[j] = t[j] >= 0 ? ldg(G + t[j]) : INF;
  }
#pragma unroll
  for (int j = 0; j < PER; ++j)
    if (t[j] >= 0 && val[j] < gt[j]) red_min(N + t[j], val[j]);
}

// Phase A. w_start/w_excl/w_val: this warp's shared scratch (32 entries each).
template <bool BIDIR>
__device__ __forceinline__ void push_local(const PushArgs& a, long long* w_start, long long* w_excl,
                                           int* w_val, int* w_src, int* w_list) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  constexpr int PER = PUSH_CHUNK / 32;
  unsigned long long work = 0;
  for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < a.nregions;
       r += nw) {
#if FSV_DELTA_GROUPS
    // expand 32 group entries at a time into this warp's vertex list (<= 128)
    const int gcnt = a.count[r];
    const int* greg = a.list + r * a.rcap;
    for (int gb = 0; gb < gcnt; gb += 32) {
    const unsigned e = gb + lane < gcnt ? (unsigned)greg[gb + lane] : 0u;
    const int nv = __popc(e & 15u);
    int vincl = nv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, vincl, o);
      if (lane >= o) vincl += y;
    }
    const int cnt = __shfl_sync(0xffffffffu, vincl, 31);
    {
      int k = vincl - nv;
      const int v0 = (int)((e >> 4) << 2);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if ((e >> j) & 1u) w_list[k++] = v0 + j;
    }
    __syncwarp();
    const int* reg = w_list;
#else
    const int cnt = a.count[r];
    const int* reg = a.list + r * a.rcap;
#endif
    for (int b = 0; b < cnt; b += 32) {
      long long deg = 0, start = 0;
      int gv = INF, vs = 0;
      if (b + lane < cnt) {
        const int v = reg[b + lane];
        vs = v;
        if (v >= a.row_begin && v < a.row_end) {
          const long long o0 = a.off[v];
          start = o0 - a.col_base;
          deg = a.off[v + 1] - o0;
          gv = ldg(a.G + v);
        }
      }
      work += (unsigned long long)deg;
      // long rows: chunk records for phase B
      unsigned big = __ballot_sync(0xffffffffu, deg > PUSH_BIG);
      while (big) {
        const int src = __ffs(big) - 1;
        big &= big - 1;
        const long long bs = __shfl_sync(0xffffffffu, start, src);
        const long long bd = __shfl_sync(0xffffffffu, deg, src);
        const int bv = __shfl_sync(0xffffffffu, gv, src);
        const int bsrc = __shfl_sync(0xffffffffu, vs, src);
        const long long nck = (bd + PUSH_BCHUNK - 1) / PUSH_BCHUNK;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(a.nchunks, (unsigned long long)nck);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (long long q = lane; q < nck; q += 32) {
          PushChunk ck;
          ck.pos_cnt = (bs + q * PUSH_BCHUNK) | (min((long long)PUSH_BCHUNK, bd - q * PUSH_BCHUNK) << 48);
          ck.val = bv;
          ck.src = bsrc;
          a.chunks[base + q] = ck;
        }
      }
      if (deg > PUSH_BIG) deg = 0;
      // short rows: flatten the batch and push it now
      long long incl = deg;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const long long T = __shfl_sync(0xffffffffu, incl, 31);
      if (T == 0) continue;
      w_start[lane] = start;
      w_excl[lane] = incl - deg;
      w_val[lane] = gv;
      w_src[lane] = vs;
      __syncwarp();
      int o = 0;   // owner of the lane's current entry (monotone in e)
      for (long long e0 = 0; e0 < T; e0 += PUSH_CHUNK) {
        int u[PER], val[PER], sv[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const long long e = e0 + lane + 32 * j;
          u[j] = -1;
          val[j] = INF;
          sv[j] = 0;
          if (e < T) {
            while (o < 31 && w_excl[o + 1] <= e) ++o;
            u[j] = ldg(a.cols + w_start[o] + (e - w_excl[o]));
            val[j] = w_val[o];
            if (BIDIR) sv[j] = w_src[o];
          }
        }
        push_entries<PER, BIDIR>(u, val, sv, a.F, a.G, a.N);
      }
      __syncwarp();
    }
#if FSV_DELTA_GROUPS
    __syncwarp();
    }
#endif
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) work += __shfl_xor_sync(0xffffffffu, work, o);
  if (lane == 0 && work) atomicAdd(a.flops, work);
}

// Phase B: one warp per long-row chunk, contiguous columns.
template <bool BIDIR>
__device__ __forceinline__ void push_big(const PushArgs& a) {
  const int lane = threadIdx.x & 31;
  const unsigned long long total = __ldcg(a.nchunks);   // written before the grid barrier (L2)
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  constexpr int PER = PUSH_BCHUNK / 32;
  for (long long q = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
       q < (long long)total; q += nw) {
    const PushChunk ck = a.chunks[q];
    const long long pos = ck.pos_cnt & ((1LL << 48) - 1);
    const int cnt = (int)(ck.pos_cnt >> 48);
    int u[PER], val[PER], sv[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int e = lane + 32 * j;
      u[j] = e < cnt ? ldg(a.cols + pos + e) : -1;
      val[j] = ck.val;
      sv[j] = ck.src;
    }
    push_entries<PER, BIDIR, true>(u, val, sv, a.F, a.G, a.N);
  }
}

// Rank-tier gather: hub slots below H from shared memory, the rest of the
// tier from the compact (L2-resident) G_hub, non-tier columns from G.
__device__ __forceinline__ int gather_gf_tier(uint32_t c, uint32_t s_base, const int* __restrict__ G,
                                              const int* __restrict__ G_hub, uint32_t H) {
  int v;
  const uint32_t x = c & IDMASK;
  const bool hub = (c & HUB) != 0;
  const bool sm = hub && x < H;
  const int* gp = hub ? G_hub + x : G + x;
#ifdef FSV_CHECKS
  if (!sm) chk_ld(gp);
#endif
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "@p  ld.shared.b32 %0, [%2];\n\t"
      "@!p ld.global.nc.b32 %0, [%3];\n\t}"
      : "=r"(v)
      : "r"((uint32_t)sm), "r"(s_base + (x << 2)), "l"(gp));
  return v;
}

// ---- phase H: hooking over the oriented layout ------------------------------
//
// Warp task = SPAN consecutive entries; lane l of a step owns entries
// [8l, 8l+8). Every entry gathers one gf value: a header its row vertex's,
// an edge its neighbour's (shared-memory hub table or global). Rows are
// contiguous, so
//   - the row open when a lane starts is the last header of the nearest lane
//     to the left that has one (one shuffle), or the step carry;
//   - row minima spanning lanes are combined by a segmented scan, and the
//     run still open at the span end is emitted as a partial (min-atomics are
//     idempotent, so partials need no fix-up).
// Fast path: an edge can only emit if its gf differs from its row's gf
// (row side needs val < gu, column side gu < val). When no entry of the step
// differs and no carried minimum is pending, the whole step is a no-op apart
// from carry bookkeeping — the common case once components have converged.

// The push over the listed vertices: phase A, grid barrier (every CTA is
// resident: one persistent CTA per SM), phase B. The scratch aliases the hub
// table in dynamic shared memory.
template <bool BIDIR>
__device__ __forceinline__ void hook_push(const HookArgs& a, int* s_hub) {
  long long* s_start = reinterpret_cast<long long*>(s_hub);
  long long* s_excl = s_start + HOOK_THREADS;
  int* s_val = reinterpret_cast<int*>(s_excl + HOOK_THREADS);
  int* s_src = s_val + HOOK_THREADS;
  int* s_list = s_src + HOOK_THREADS;            // 128 expanded vertices per warp
  const int wib = threadIdx.x >> 5;
  DBG_T(0);
  push_local<BIDIR>(a.push, s_start + wib * 32, s_excl + wib * 32, s_val + wib * 32, s_src + wib * 32,
                    s_list + wib * 128);
  __syncthreads();
  DBG_T(1);
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(a.push.barrier, 1u);
    while (*(volatile unsigned*)a.push.barrier < gridDim.x) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
  DBG_T(2);
  push_big<BIDIR>(a.push);
#ifdef FSV_DEBUG_TIMING
  __syncthreads();
  DBG_T(3);
#endif
}

// Minority sweep of a dense iteration. Once one component dominates, almost
// every vertex carries the same grandparent r, and an entry can only
// contribute when its endpoints' gf differ, i.e. when at least one endpoint
// is outside that majority. So instead of sweeping every stored entry, list
// the vertices with gf != r (r = gf of the most connected vertex, hub slot
// 0) and push along their symmetric CSR rows in both directions: gf[x] to a
// neighbour y with a larger gf, and gf[y] back into N[x] when it is smaller
// (an edge between two listed vertices is visited twice, which a min
// absorbs). This is the same set of aggressive hooks as the dense sweep
// makes; the stochastic ones follow in the vertex pass either way. The lists
// go into the vertex pass's delta regions (free during a dense hook, same
// 4-vertex group format), with the degree sum of the listed vertices; all
// CTAs then take the same branch: the push if the sum is at most
// minority_thr, else the dense sweep. Across ranks the gf vector and the row
// offsets are replicated, so every rank lists the same vertices, computes
// the same sum and takes the same branch, and pushes only from the listed
// vertices of its own rows (each edge at a listed vertex is then visited by
// the rank that owns that vertex's row). Returns true when the iteration is
// done.
__device__ __forceinline__ bool hook_minority(const HookArgs& a, int* s_hub, int r, unsigned long long* mdeg,
                                              unsigned* mbar) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long n4 = a.n >> 2, ngroups = (a.n + 3) >> 2;
  const int nreg = a.push.nregions;
  const long long gper = (ngroups + nreg - 1) / nreg;          // groups per region (<= rcap, see upload_impl)
  const int4* G4 = reinterpret_cast<const int4*>(a.G);
  unsigned long long dsum = 0;
  for (int w = gw; w < nreg; w += nwarps) {
    int* region = a.mlist + (long long)w * a.push.rcap;
    int wo = 0;
    const long long g0 = w * gper, g1 = min(g0 + gper, ngroups);
    for (long long gb = g0; gb < g1; gb += 32) {
      const long long g = gb + lane;
      unsigned m4 = 0;
      if (g < g1) {
        // the group's gf values and degrees from vector loads; vertices
        // without edges (most of a skewed graph's minority) are not listed
        long long d0, d1, d2, d3;
        if (g < n4) {
          const int4 v = G4[g];
          m4 = (v.x != r) | ((v.y != r) << 1) | ((v.z != r) << 2) | ((v.w != r) << 3);
          if (a.off32) {
            const int4 o = reinterpret_cast<const int4*>(a.off32)[g];
            const int o4 = a.off32[(g << 2) + 4];
            d0 = o.y - o.x; d1 = o.z - o.y; d2 = o.w - o.z; d3 = o4 - o.w;
          } else {
            const longlong2 oa = reinterpret_cast<const longlong2*>(a.push.off)[2 * g];
            const longlong2 ob = reinterpret_cast<const longlong2*>(a.push.off)[2 * g + 1];
            const long long o4 = a.push.off[(g << 2) + 4];
            d0 = oa.y - oa.x; d1 = ob.x - oa.y; d2 = ob.y - ob.x; d3 = o4 - ob.y;
          }
        } else {
          d0 = d1 = d2 = d3 = 0;
          for (int j = 0; j < (int)(a.n & 3); ++j) {
            const long long v = (g << 2) + j;
            m4 |= (a.G[v] != r ? 1u : 0u) << j;
            const long long d = a.push.off[v + 1] - a.push.off[v];
            if (j == 0) d0 = d; else if (j == 1) d1 = d; else d2 = d;
          }
        }
        m4 &= (d0 > 0 ? 1u : 0u) | (d1 > 0 ? 2u : 0u) | (d2 > 0 ? 4u : 0u) | (d3 > 0 ? 8u : 0u);
        dsum += (unsigned long long)(((m4 & 1u) ? d0 : 0) + ((m4 & 2u) ? d1 : 0) + ((m4 & 4u) ? d2 : 0) +
                                     ((m4 & 8u) ? d3 : 0));
      }
      const bool on = m4 != 0u;
      const unsigned bal = __ballot_sync(0xffffffffu, on);
      if (on) region[wo + __popc(bal & lt)] = (int)(((unsigned)g << 4) | m4);
      wo += __popc(bal);
    }
    if (lane == 0) a.mcount[w] = wo;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
  if (lane == 0 && dsum) atomicAdd(mdeg, dsum);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(mbar, 1u);
    while (*(volatile unsigned*)mbar < gridDim.x) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
#ifdef FSV_DEBUG_MINORITY
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("[minority] iter %d r %d degree sum %llu thr %lld\n", a.iter, r, __ldcg(mdeg), a.minority_thr);
#endif
  if ((long long)__ldcg(mdeg) > a.minority_thr) return false;
  if (blockIdx.x == 0 && threadIdx.x == 0) mdeg[C_MDONE - C_MDEG] = 1ull;
  hook_push<true>(a, s_hub);
  return true;
}

// HUBS = false (no hub slots, H == 0) compiles the hub table, hub mask and
// accumulators out; TIER (implies HUBS) adds the L2 rank tier gathers.
template <bool HUBS, bool TIER, int NSTEP>
__global__ void __launch_bounds__(HOOK_THREADS, 1) k_hook(HookArgs a) {
  extern __shared__ int s_hub[];
  if (__ldcg(a.done)) return;
  if (a.lc.graph == 1) {
    const int it = loop_iter(a.lc, a.iter);
    unsigned long long* slot = a.lc.cnt_base + (size_t)(it - 1) * NCOUNT;
    a.iter = it;
    a.push.iter = it;
    int *Fb, *Nb;
    loop_bufs(a.lc, it, Fb, Nb);
    a.F = Fb; a.N = Nb; a.push.F = Fb; a.push.N = Nb;
    a.push.flops = slot + C_FLOPS;
    a.push.nchunks = slot + C_CHUNKS;
    a.push.barrier = reinterpret_cast<unsigned*>(slot + C_BARRIER);
    a.fix_barrier = reinterpret_cast<unsigned*>(slot + C_FIXBAR);
    a.task_ctr = reinterpret_cast<unsigned*>(slot + C_SPANS);
  }
  if (a.mode[a.iter] == 1) {
    hook_push<false>(a, s_hub);   // sparse iteration: push from the vertices whose gf changed
    return;
  }
  if (HUBS && a.minority_thr >= 0 && a.iter >= 3) {
    // (iteration 2 follows the closed-form first iteration: no majority yet)
    unsigned long long* slot = a.lc.cnt_base + (size_t)(a.iter - 1) * NCOUNT;
    if (hook_minority(a, s_hub, __ldcg(a.G_hub), slot + C_MDEG, reinterpret_cast<unsigned*>(slot + C_MBAR)))
      return;
  }
  // s_hub[0, HOT_ACC): this CTA's accumulator of the hottest hub slots;
  // s_hub[HOT_ACC, HOT_ACC + H): gf of the shared-memory hubs. Both bases are
  // constants, so neither costs a register in the loop. Only slots < HT ever
  // receive a value, so both passes over the accumulator run to HOT_ACC.
  if (HUBS) {
    for (int i = threadIdx.x; i < (a.H >> 2); i += blockDim.x)
      reinterpret_cast<int4*>(s_hub + HOT_ACC)[i] = reinterpret_cast<const int4*>(a.G_hub)[i];
    for (int i = threadIdx.x; i < HOT_ACC; i += blockDim.x) s_hub[i] = INF;
    __syncthreads();
  }
  const uint32_t s_acc = (uint32_t)__cvta_generic_to_shared(s_hub);
  const uint32_t s_base = s_acc + 4u * HOT_ACC;

  const int* __restrict__ G = a.G;
  int* __restrict__ N = a.N;
  int* __restrict__ hub_acc = a.hub_acc;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  // span counts fit 32 bits (2^31 spans = 2^41 entries); a 64-bit counter
  // costs a register the loop body cannot spare
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nspans = (int)a.nspans;
  const uint64_t pol = policy_evict_first();

  bool dense = false;   // warp-uniform, see FSV_DENSE_LANES
  // Tasks gw, gw + nwarps, ... for the first `fixed` rounds, then (hub-table
  // kernels with at least 4 rounds, FSV_DYN_TAIL > 0) one task at a time
  // from a shared counter: the slow warps of a launch no longer set its tail,
  // which every CTA waits out at the hub fix-up barrier.
  const int rounds = nspans / nwarps;
  constexpr bool DYN = FSV_DYN_TAIL > 0 && (HUBS || FSV_DYN_NOHUB);
  const int fixed = (DYN && rounds >= 4) ? rounds - FSV_DYN_TAIL : INF;
  int k = 0;
  for (int s = gw; s < nspans;) {
    int carry_u = ldg(a.span_row + s);              // row open at the task start
    int carry_gu = carry_u >= 0 ? ldg(G + carry_u) : INF;
    int carry_run = INF;
    const uint4* p = reinterpret_cast<const uint4*>(a.ecol + (size_t)s * (NSTEP * STEP)) + 2 * lane;
    Entries8 nx = ld_stream8(p, pol);
#pragma unroll 1
    for (int st = 0; st < NSTEP; ++st) {
      const uint32_t c[EPL] = {nx.c[0], nx.c[1], nx.c[2], nx.c[3], nx.c[4], nx.c[5], nx.c[6], nx.c[7]};
      if (st + 1 < NSTEP) {
        nx = ld_stream8(p + (st + 1) * 64, pol);
      }
      int val[EPL];
#pragma unroll
      for (int j = 0; j < EPL; ++j)
#if FSV_SOL & 2
        val[j] = s_hub[HOT_ACC + (c[j] & 0x7fffu)];   // dev speed-of-light probe: no global gathers (wrong results)
#else
        val[j] = TIER ? gather_gf_tier(c[j], s_base, G, a.G_hub, (uint32_t)a.H)
                      : gather_gf(c[j], s_base, G);
#endif
      // last header of this lane
      int lu = -1, lgu = INF;
#pragma unroll
      for (int j = 0; j < EPL; ++j)
        if ((int)c[j] < 0) { lu = (int)(c[j] & IDMASK); lgu = val[j]; }
      const unsigned hb = __ballot_sync(0xffffffffu, lu >= 0);
      const unsigned left = hb & lt;
      const int src = left ? 31 - __clz(left) : lane;
      int in_u = __shfl_sync(0xffffffffu, lu, src);
      int in_gu = __shfl_sync(0xffffffffu, lgu, src);
      if (!left) { in_u = carry_u; in_gu = carry_gu; }
      // Entries that differ from their row's gf, as per-entry records
      // (target, value): val < gf(row) is a row-side contribution to the row
      // vertex, val > gf(row) a column-side one to the neighbour (or its hub
      // slot). At most FSV_REC records per lane are kept in registers.
      // (skipped while the warp is in dense mode: the last scan step had
      // emissions on most lanes, so the next one almost surely needs the scan)
      int nrec = 0;
      if (!dense) {
        int rg = in_gu;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          rg = ((int)c[j] < 0) ? val[j] : rg;
          nrec += (val[j] != rg) ? 1 : 0;   // never for a header
        }
      }
      if (!dense && !__any_sync(0xffffffffu, nrec > 0) && carry_run >= carry_gu) {
        if (hb) {
          const int last = 31 - __clz(hb);
          carry_u = __shfl_sync(0xffffffffu, lu, last);
          carry_gu = __shfl_sync(0xffffffffu, lgu, last);
          carry_run = INF;
        }
        continue;
      }
#if FSV_REC > 0
      // ---- record path: few differing entries ------------------------------
      // Each differing entry is emitted on its own (min-atomics are
      // idempotent, so a row minimum may arrive as several partial minima;
      // the smallest of them is the row minimum). No scan, no pending run:
      // a run carried in from a scan step is emitted here by lane 0.
      if (!dense && !__any_sync(0xffffffffu, nrec > FSV_REC)) {
        if (lane == 0) emit_agg(carry_u, carry_gu, carry_run, N);
        if (nrec && !(FSV_SOL & 1)) {
          // second pass: pick out the (at most two) records of this lane
          uint32_t rx0 = 0u, rx1 = 0u;
          int ry0 = 0, ry1 = 0;
          {
            int rg = in_gu, ru = in_u, k = 0;
#pragma unroll
            for (int j = 0; j < EPL; ++j) {
              const bool h = (int)c[j] < 0;
              rg = h ? val[j] : rg;
              ru = h ? (int)(c[j] & IDMASK) : ru;
              const bool d = val[j] != rg;
              const bool rs = val[j] < rg;
              const uint32_t xr = rs ? (uint32_t)ru : c[j];
              const int yr = rs ? val[j] : rg;
              if (d && k == 0) { rx0 = xr; ry0 = yr; }
              if (d && k == 1) { rx1 = xr; ry1 = yr; }
              k += d ? 1 : 0;
            }
          }
          const bool h0 = HUBS && (rx0 & HUB), h1 = HUBS && nrec > 1 && (rx1 & HUB);
          const bool g1 = nrec > 1 && !h1;
          const int x0 = (int)(rx0 & IDMASK), x1 = (int)(rx1 & IDMASK);
          if (h0) {
            if (x0 < HOT_ACC) red_min_shared(s_acc + 4u * (uint32_t)x0, ry0);
            else red_min(hub_acc + acc_idx<TIER>(x0), ry0);
          } else {
            red_min(N + x0, ry0);
          }
          if (h1) {
            if (x1 < HOT_ACC) red_min_shared(s_acc + 4u * (uint32_t)x1, ry1);
            else red_min(hub_acc + acc_idx<TIER>(x1), ry1);
          } else if (g1) {
            red_min(N + x1, ry1);
          }
        }
        carry_run = INF;
        if (hb) {
          const int last = 31 - __clz(hb);
          carry_u = __shfl_sync(0xffffffffu, lu, last);
          carry_gu = __shfl_sync(0xffffffffu, lgu, last);
        }
        continue;
      }
#endif
      // ---- slow path ------------------------------------------------------
      // One emission slot per entry, filled branch-free:
      //   header j: closes the row before it (the lane's first header closes
      //             the row entering the lane; handled after the scan)
      //             target = previous row vertex, value = its run min,
      //             threshold = its gf
      //   edge j:   column side, target = v (or hub slot), value = row gf,
      //             threshold = gf[v]
      // then every active slot does N[target] <-min value (the stochastic
      // N[F[target]] <-min value is deferred to the vertex pass).
      int cu = in_u, cgu = in_gu, run = INF, pre = INF;
      bool seen = false;
      unsigned act = 0, hubm = 0;
      int w[EPL], y[EPL];
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        const bool h = (int)c[j] < 0;
        const bool first = h && !seen;
        pre = first ? run : pre;
        const int yj = h ? run : cgu;
        const int gj = h ? cgu : val[j];
        w[j] = h ? cu : (int)(c[j] & IDMASK);
        y[j] = yj;
        act |= ((yj < gj) && !first ? 1u : 0u) << j;
        if (HUBS) hubm |= (!h && (c[j] & HUB) ? 1u : 0u) << j;
        seen |= h;
        cu = h ? (int)(c[j] & IDMASK) : cu;
        cgu = h ? val[j] : cgu;
        run = h ? INF : min(run, val[j]);
      }
      if (act && !(FSV_SOL & 1)) {
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          if ((act >> j) & 1u) {
            if (HUBS && ((hubm >> j) & 1u)) {
              if (w[j] < HOT_ACC) red_min_shared(s_acc + 4u * (uint32_t)w[j], y[j]);
              else red_min(hub_acc + acc_idx<TIER>(w[j]), y[j]);
            } else {
              red_min(N + w[j], y[j]);
            }
          }
        }
      }
#if FSV_DENSE_LANES > 0
      if (HUBS) dense = __popc(__ballot_sync(0xffffffffu, act != 0)) >= FSV_DENSE_LANES;
#endif
      // segmented inclusive scan of (seen, run): min of the run open at the
      // end of each lane
      int sv = run, sf = seen ? 1 : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int ov = __shfl_up_sync(0xffffffffu, sv, off);
        const int of = __shfl_up_sync(0xffffffffu, sf, off);
        if (lane >= off) { if (!sf) sv = min(sv, ov); sf |= of; }
      }
      const int ev = __shfl_up_sync(0xffffffffu, sv, 1);
      const int ef = __shfl_up_sync(0xffffffffu, sf, 1);
      const int cin = (lane == 0) ? carry_run : (ef ? ev : min(ev, carry_run));
      if (seen) {
        const int v = min(cin, pre);
        if (v < in_gu) red_min(N + in_u, v);  // row entering the lane closes here
      }
      const int lv = __shfl_sync(0xffffffffu, sv, 31);
      const int lf = __shfl_sync(0xffffffffu, sf, 31);
      carry_run = lf ? lv : min(lv, carry_run);
      if (hb) {
        const int last = 31 - __clz(hb);
        carry_u = __shfl_sync(0xffffffffu, lu, last);
        carry_gu = __shfl_sync(0xffffffffu, lgu, last);
      }
    }
    // the run still open at the span end: partial minimum of row carry_u
    if (lane == 0) emit_agg(carry_u, carry_gu, carry_run, N);
    if constexpr (DYN) {
      if (++k < fixed) {
        s += nwarps;
      } else {
        unsigned q = 0;
        if (lane == 0) q = atomicAdd(a.task_ctr, 1u);
        s = fixed * nwarps + (int)__shfl_sync(0xffffffffu, q, 0);
      }
    } else {
      s += nwarps;
    }
  }
  if (HUBS) {
    __syncthreads();
    for (int i = threadIdx.x; i < HOT_ACC; i += blockDim.x) {
      const int v = s_hub[i];
      if (v != INF) red_min(hub_acc + (long long)i * FSV_ACC_STRIDE, v);   // (HOT_ACC <= ACC_SPREAD)
    }
#if FSV_FUSE_HUBFIX
    // hub fix-up in the same launch: grid barrier (every CTA is resident),
    // then the accumulated column-side minima go to N (k_hubfix's work)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(a.fix_barrier, 1u);
      while (*(volatile unsigned*)a.fix_barrier < gridDim.x) __nanosleep(32);
      __threadfence();
    }
    __syncthreads();
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < a.HT; s += gridDim.x * blockDim.x) {
      const int acc = __ldcg(hub_acc + acc_at(s));
      if (acc == INF) continue;
      hub_acc[acc_at(s)] = INF;
      emit_agg(ldg(a.hub_id + s), ldg(a.G_hub + s), acc, N);
    }
#endif
  }
}

// ---- hub accumulator -> N ---------------------------------------------------

// gf of slot s is G_hub[s] (compact, refreshed by the vertex pass), not a
// random gather of G[hub_id[s]].
__global__ void k_hubfix(int* __restrict__ hub_acc, const int* __restrict__ hub_id,
                         const int* __restrict__ G_hub, int H, int* __restrict__ N, const int* done,
                         const int* mode, int iter, const int* iterp, int* X, int* Y) {
  if (__ldcg(done)) return;
  if (iterp) {   // graph mode: iteration and buffers from the device (loop_bufs)
    iter = __ldcg(iterp);
    N = (iter & 1) ? Y : X;
  }
  if (mode[iter] != 0) return;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < H; s += gridDim.x * blockDim.x) {
    const int acc = hub_acc[acc_at(s)];
    if (acc == INF) continue;
    hub_acc[acc_at(s)] = INF;
    const int h = ldg(hub_id + s);
    emit_agg(h, ldg(G_hub + s), acc, N);
  }
}

// ---- counters + convergence flag --------------------------------------------
// Each block writes its five partial counts; the last block to finish (ticket)
// sums them, stores this iteration's counters and raises the convergence flag
// when gf did not change. No same-address atomics besides the ticket.

template <int NT>
__device__ __forceinline__ void finish_counters(const unsigned (&c)[5], unsigned* partials,
                                                unsigned long long* cnt, unsigned int* ticket,
                                                int* done, int iter, int max_iter,
                                                const DeltaOut& dl, const LoopCtl& lc) {
  __shared__ unsigned s_part[NT / 32][5];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const unsigned v = __reduce_add_sync(0xffffffffu, c[k]);
    if (lane == 0) s_part[w][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    unsigned sum = 0;
    for (int i = 0; i < NT / 32; ++i) sum += s_part[i][threadIdx.x];
    partials[(size_t)blockIdx.x * 8 + threadIdx.x] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  unsigned long long acc[5] = {0ull, 0ull, 0ull, 0ull, 0ull};
  for (unsigned b = threadIdx.x; b < gridDim.x; b += NT) {
#pragma unroll
    for (int k = 0; k < 5; ++k) acc[k] += __ldcg(partials + (size_t)b * 8 + k);
  }
  __shared__ unsigned long long s_acc[NT / 32][5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    unsigned long long v = acc[k];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_acc[w][k] = v;
  }
  __syncthreads();
  __shared__ int s_stop;
  if (threadIdx.x < 5) {
    unsigned long long sum = 0;
    for (int i = 0; i < NT / 32; ++i) sum += s_acc[i][threadIdx.x];
    cnt[threadIdx.x] = sum;
    if (threadIdx.x == C_GF) {
      bool stop = true;
      if (sum == 0ull) atomicExch(done, iter);
      else if (max_iter > 0 && iter >= max_iter) atomicExch(done, -iter);
      else stop = false;
      s_stop = stop ? (sum == 0ull ? iter : -iter) : 0;
      lc.tstamp[iter] = global_ns();
      if (lc.graph) *lc.iterp = iter + 1;                       // 2: iteration 1 before the graph
      if (lc.graph == 1) {
        cudaGraphSetConditional(lc.cond, stop ? 0u : 1u);
        if (lc.cond_next) cudaGraphSetConditional(lc.cond_next, stop ? 0u : 1u);
      }
      // product choice for the next iteration (choose_kernel, driver.py:51-61)
      int m = 0;
      if (dl.policy == 2) m = 1;
      else if (dl.policy == 0) m = ((double)sum < dl.threshold * (double)dl.n_total) ? 1 : 0;
      dl.mode[iter + 1] = m;
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;
  if (lc.rep) {
    // the final iteration packs the solve's report for a single host copy
    __syncthreads();
    const int fin = s_stop;
    if (fin) {
      const int it = fin > 0 ? fin : -fin;
      const int k = it <= STAGE_ITERS ? it : 0;
      for (int i = threadIdx.x; i < k * NCOUNT; i += NT) lc.rep->cnt[i] = __ldcg(lc.cnt_base + i);
      if (k)
        for (int i = threadIdx.x; i <= k + 1; i += NT) lc.rep->mode[i] = __ldcg(lc.mode_base + i);
      if (k)
        for (int i = threadIdx.x; i <= k; i += NT) lc.rep->ts[i] = __ldcg(lc.tstamp + i);
      if (threadIdx.x == 0) {
        lc.rep->iters = k;
        lc.rep->done = fin;
      }
    }
  }
}

// ---- phase G: grandparents, counters, next N init ---------------------------

// Append the vertices u0+j (j < 4, bit j of m4) to this warp's delta region.
#if FSV_DELTA_GROUPS
// Delta entries are 4-vertex groups: (u0/4) << 4 | bit mask of the changed
// vertices among u0..u0+3 (one ballot per group instead of one per vertex);
// the push expands them.
__device__ __forceinline__ void delta_append(unsigned m4, int u0, int* region, int& wo) {
  const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
  const bool on = m4 != 0u;
  const unsigned b = __ballot_sync(0xffffffffu, on);
  if (on) region[wo + __popc(b & lt)] = (int)((((unsigned)u0 >> 2) << 4) | m4);
  wo += __popc(b);
}
#else
__device__ __forceinline__ void delta_append(unsigned m4, int u0, int* region, int& wo) {
  const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool on = (m4 >> j) & 1u;
    const unsigned b = __ballot_sync(0xffffffffu, on);
    if (on) region[wo + __popc(b & lt)] = u0 + j;
    wo += __popc(b);
  }
}
#endif

// Vertex pass of iteration k >= 2 over groups of 4 consecutive vertices
// (int4 index i): gf' = N[N], counters, next N init, delta append. Loads of
// both groups a thread owns are issued before any store or ballot so their
// latencies overlap. `valid` = false lanes only take part in the ballots.
struct SGroup {
  int4 nu, go, fo, gg;
};

__device__ __forceinline__ void sgroup_load(bool valid, long long i, const int4* N4,
                                            const int* __restrict__ N, const int4* F4,
                                            const int4* G4, SGroup& g) {
  if (valid) {
    g.nu = N4[i];
    g.go = G4[i];
    g.fo = F4[i];
    g.gg.x = ldg(N + g.nu.x); g.gg.y = ldg(N + g.nu.y);
    g.gg.z = ldg(N + g.nu.z); g.gg.w = ldg(N + g.nu.w);
  }
}

__device__ __forceinline__ void sgroup_commit(bool valid, long long i, const SGroup& g, int4* F4,
                                              int4* G4, unsigned (&c)[5], int* region, int& wo) {
  unsigned m4 = 0;
  if (valid) {
    const int u = (int)(i << 2);
    const int4 nu = g.nu, go = g.go, fo = g.fo, gg = g.gg;
    c[C_GF] += (gg.x != go.x) + (gg.y != go.y) + (gg.z != go.z) + (gg.w != go.w);
    c[C_F] += (nu.x != fo.x) + (nu.y != fo.y) + (nu.z != fo.z) + (nu.w != fo.w);
    c[C_NONSTAR] += (gg.x != nu.x) + (gg.y != nu.y) + (gg.z != nu.z) + (gg.w != nu.w);
    c[C_ROOTS] += (nu.x == u) + (nu.y == u + 1) + (nu.z == u + 2) + (nu.w == u + 3);
    c[C_VIOL] += (nu.x > fo.x) + (nu.y > fo.y) + (nu.z > fo.z) + (nu.w > fo.w);
    m4 = (gg.x != go.x) | ((gg.y != go.y) << 1) | ((gg.z != go.z) << 2) | ((gg.w != go.w) << 3);
    // stores only where the value changes: once most vertices are stable,
    // whole sectors stay clean and are never written back to DRAM
    if (m4) G4[i] = gg;
    if ((gg.x != fo.x) | (gg.y != fo.y) | (gg.z != fo.z) | (gg.w != fo.w)) F4[i] = gg;
  }
  delta_append(m4, (int)(i << 2), region, wo);
}

// Scalar tail (n % 4 vertices), run by warp 0 lanes 0..2 after the vector part.
template <typename Fn>
__device__ __forceinline__ void tail_append(long long n4, long long n, Fn&& one, int* region, int& wo) {
  const long long u = (n4 << 2) + (threadIdx.x & 31);
  const bool ch = (u < n) ? one(u) : false;
  const unsigned b = __ballot_sync(0xffffffffu, ch);
#if FSV_DELTA_GROUPS
  // the tail (< 4 vertices) is group n4; lanes 0..2 hold its vertices
  if ((threadIdx.x & 31) == 0 && b) region[wo] = (int)(((unsigned)n4 << 4) | (b & 15u));
  wo += b ? 1 : 0;
#else
  if (ch) region[wo + __popc(b & ((1u << (threadIdx.x & 31)) - 1u))] = (int)u;
  wo += __popc(b);
#endif
}

#ifndef FSV_SC_MINB
#define FSV_SC_MINB 2
#endif
__global__ void __launch_bounds__(SC_THREADS, FSV_SC_MINB) k_shortcut(ShortcutArgs a) {
  if (converged_exit(a.done, a.lc)) return;
  if (a.lc.graph == 1) {
    a.iter = loop_iter(a.lc, a.iter);
    a.cnt = a.lc.cnt_base + (size_t)(a.iter - 1) * NCOUNT;
    int* Nb;
    loop_bufs(a.lc, a.iter, a.F, Nb);
    a.N = Nb;
  }
  unsigned c[5] = {0u, 0u, 0u, 0u, 0u};
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const long long n4 = a.n >> 2;
  int4* F4 = reinterpret_cast<int4*>(a.F);
  int4* G4 = reinterpret_cast<int4*>(a.G);
  const int4* N4 = reinterpret_cast<const int4*>(a.N);
  if (a.mode[a.iter] == 0) {
    // Stochastic hooks of a dense iteration. The sweep only applied the
    // aggressive hooks, so N[u] = min(gf[u], mngf[u]) here; a vertex it
    // lowered (N[u] < gf[u], hence N[u] = mngf[u]) now hooks its parent:
    // f[f_k[u]] <-min mngf[u] (kernels.py:110-118). BSP: every mngf[u] must
    // be read before any N is lowered here, so pass A parks the lowered
    // vertices' values (in registers, or in G with the sign bit set: G[u] is
    // only read by its own thread until the final pass rewrites it, since a
    // lowered vertex's gf always changes), a grid barrier follows (all blocks
    // are resident: cooperative launch), pass B issues the reductions, and a
    // second barrier precedes the grandparent gathers below.
    // The first PARK groups of a thread stay in registers (every group when
    // n <= 4 * PARK * threads, e.g. RMAT-22); only the rest go through G.
    constexpr int PARK = 8;
    int4 pk[PARK];
#pragma unroll
    for (int j = 0; j < PARK; ++j) {
      const long long i = t0 + j * stride;
      pk[j] = make_int4(-1, -1, -1, -1);
      if (i < n4) {
        int4 nu;   // (L2 load: the final pass must not find a stale copy in L1)
        asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(nu.x), "=r"(nu.y), "=r"(nu.z), "=r"(nu.w) : "l"(N4 + i));
        const int4 go = G4[i];
        pk[j].x = nu.x < go.x ? nu.x : -1;
        pk[j].y = nu.y < go.y ? nu.y : -1;
        pk[j].z = nu.z < go.z ? nu.z : -1;
        pk[j].w = nu.w < go.w ? nu.w : -1;
      }
    }
    unsigned touched = 0;   // bit j: the thread's (PARK + j)-th group holds a lowered vertex (j >= 31 share bit 31)
    int j = 0;
    for (long long i = t0 + PARK * stride; i < n4; i += stride, ++j) {
      int4 nu;
      asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(nu.x), "=r"(nu.y), "=r"(nu.z), "=r"(nu.w) : "l"(N4 + i));
      int4 go = G4[i];
      const bool lx = nu.x < go.x, ly = nu.y < go.y, lz = nu.z < go.z, lw = nu.w < go.w;
      if (lx | ly | lz | lw) {
        if (lx) go.x = nu.x | (int)0x80000000;
        if (ly) go.y = nu.y | (int)0x80000000;
        if (lz) go.z = nu.z | (int)0x80000000;
        if (lw) go.w = nu.w | (int)0x80000000;
        G4[i] = go;
        touched |= 1u << min(j, 31);
      }
    }
    int tail_val = -1;   // the scalar tail (n % 4 vertices): its values stay in a register
    if (t0 < (a.n & 3)) {
      const long long u = (n4 << 2) + t0;
      const int nu = __ldcg(a.N + u);
      if (nu < a.G[u]) tail_val = nu;
    }
    unsigned* bar = reinterpret_cast<unsigned*>(a.cnt + C_SCBAR);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(bar, 1u);
      while (*(volatile unsigned*)bar < gridDim.x) __nanosleep(32);
      __threadfence();
    }
    __syncthreads();
#pragma unroll
    for (int j2 = 0; j2 < PARK; ++j2) {
      const int4 v = pk[j2];
      if ((v.x & v.y & v.z & v.w) < 0) continue;   // all -1: nothing lowered in this group
      const long long i = t0 + j2 * stride;
      const int4 fo = F4[i];
      const int u = (int)(i << 2);
      if (v.x >= 0 && fo.x != u) red_min(a.N + fo.x, v.x);
      if (v.y >= 0 && fo.y != u + 1) red_min(a.N + fo.y, v.y);
      if (v.z >= 0 && fo.z != u + 2) red_min(a.N + fo.z, v.z);
      if (v.w >= 0 && fo.w != u + 3) red_min(a.N + fo.w, v.w);
    }
    j = 0;
    for (long long i = t0 + PARK * stride; i < n4; i += stride, ++j) {
      if (!((touched >> min(j, 31)) & 1u)) continue;
      const int4 go = G4[i], fo = F4[i];
      const int u = (int)(i << 2);
      if (go.x < 0 && fo.x != u) red_min(a.N + fo.x, go.x & 0x7fffffff);
      if (go.y < 0 && fo.y != u + 1) red_min(a.N + fo.y, go.y & 0x7fffffff);
      if (go.z < 0 && fo.z != u + 2) red_min(a.N + fo.z, go.z & 0x7fffffff);
      if (go.w < 0 && fo.w != u + 3) red_min(a.N + fo.w, go.w & 0x7fffffff);
    }
    if (tail_val >= 0) {
      const long long u = (n4 << 2) + t0;
      const int fo = a.F[u];
      if (fo != (int)u) red_min(a.N + fo, tail_val);
    }
    bar = reinterpret_cast<unsigned*>(a.cnt + C_SCBAR2);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(bar, 1u);
      while (*(volatile unsigned*)bar < gridDim.x) __nanosleep(32);
      __threadfence();
    }
    __syncthreads();
  }
  const int* __restrict__ N = a.N;
  // warp gw handles groups [wb, wb+32) of every stride: its delta region is private
  const long long gwarp = t0 >> 5;
  int* region = a.dl.list + gwarp * a.dl.rcap;
  int wo = 0;
  for (long long wb = t0 - lane; wb < n4; wb += 2 * stride) {   // warp-uniform bound
    const long long i0 = wb + lane, i1 = wb + stride + lane;     // two groups in flight
    SGroup g0, g1;
    sgroup_load(i0 < n4, i0, N4, N, F4, G4, g0);
    sgroup_load(i1 < n4, i1, N4, N, F4, G4, g1);
    sgroup_commit(i0 < n4, i0, g0, F4, G4, c, region, wo);
    sgroup_commit(i1 < n4, i1, g1, F4, G4, c, region, wo);
  }
  if (gwarp == 0)
    tail_append(n4, a.n, [&](long long u) {
      const int nu = N[u], go = a.G[u], fo = a.F[u];
      const int gg = ldg(N + nu);
      c[C_GF] += gg != go; c[C_F] += nu != fo; c[C_NONSTAR] += gg != nu;
      c[C_ROOTS] += nu == (int)u; c[C_VIOL] += nu > fo;
      a.G[u] = gg; a.F[u] = gg;
      return gg != go;
    }, region, wo);
  if (lane == 0) a.dl.count[gwarp] = wo;
  for (long long s = t0; s < a.H; s += stride) {
    const int h = ldg(a.hub_id + s);
    a.G_hub[s] = ldg(N + ldg(N + h));
  }
  finish_counters<SC_THREADS>(c, a.partials, a.cnt, a.ticket, a.done, a.iter, a.max_iter, a.dl, a.lc);
}

// ---- iteration 1 in closed form ---------------------------------------------
// f_1[u] = min(u, min neighbour) = f1[u]; gf_1 = f1[f1]. f_1 stays in f1's
// buffer (it is the Y parent buffer); writes G = gf_1 and X = gf_1 (the N
// init of iteration 2).
struct FirstArgs {
  const int* f1;
  int* G;
  int* X;
  long long n;
  const int* hub_id;
  int* G_hub;
  int H;
  unsigned long long* cnt;
  unsigned* partials;
  unsigned int* ticket;
  int* done;
  int max_iter;
  DeltaOut dl;
  LoopCtl lc;
};

__global__ void __launch_bounds__(SC_THREADS) k_first(FirstArgs a) {
  unsigned c[5] = {0u, 0u, 0u, 0u, 0u};
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const long long n4 = a.n >> 2;
  const int* __restrict__ f1 = a.f1;
  const int4* f14 = reinterpret_cast<const int4*>(f1);
  const long long gwarp = t0 >> 5;
  int* region = a.dl.list + gwarp * a.dl.rcap;
  int wo = 0;
  for (long long wb = t0 - lane; wb < n4; wb += stride) {
    const long long i = wb + lane;
    unsigned m4 = 0;
    if (i < n4) {
      const int4 f = f14[i];
      int4 gg;
      gg.x = ldg(f1 + f.x); gg.y = ldg(f1 + f.y); gg.z = ldg(f1 + f.z); gg.w = ldg(f1 + f.w);
      const int u = (int)(i << 2);
      c[C_GF] += (gg.x != u) + (gg.y != u + 1) + (gg.z != u + 2) + (gg.w != u + 3);
      c[C_F] += (f.x != u) + (f.y != u + 1) + (f.z != u + 2) + (f.w != u + 3);
      c[C_NONSTAR] += (gg.x != f.x) + (gg.y != f.y) + (gg.z != f.z) + (gg.w != f.w);
      c[C_ROOTS] += (f.x == u) + (f.y == u + 1) + (f.z == u + 2) + (f.w == u + 3);
      c[C_VIOL] += (f.x > u) + (f.y > u + 1) + (f.z > u + 2) + (f.w > u + 3);
      reinterpret_cast<int4*>(a.G)[i] = gg;
      reinterpret_cast<int4*>(a.X)[i] = gg;
      m4 = (gg.x != u) | ((gg.y != u + 1) << 1) | ((gg.z != u + 2) << 2) | ((gg.w != u + 3) << 3);
    }
    delta_append(m4, (int)(i << 2), region, wo);
  }
  if (gwarp == 0)
    tail_append(n4, a.n, [&](long long u) {
      const int f = f1[u];
      const int gg = ldg(f1 + f);
      c[C_GF] += gg != (int)u; c[C_F] += f != (int)u; c[C_NONSTAR] += gg != f;
      c[C_ROOTS] += f == (int)u; c[C_VIOL] += f > (int)u;
      a.G[u] = gg; a.X[u] = gg;
      return gg != (int)u;
    }, region, wo);
  if (lane == 0) a.dl.count[gwarp] = wo;
  for (long long s = t0; s < a.H; s += stride) {
    const int h = ldg(a.hub_id + s);
    a.G_hub[s] = ldg(f1 + ldg(f1 + h));
  }
  finish_counters<SC_THREADS>(c, a.partials, a.cnt, a.ticket, a.done, 1, a.max_iter, a.dl, a.lc);
}

// ---- solve-start initialisation ----------------------------------------------
__global__ void k_solve_init(int* X, int* Y, int* G, long long n, int* hub_acc, int H,
                             unsigned long long* cnt, long long ncnt, int* done, unsigned* ticket,
                             int* mode, int first_mode, unsigned long long* tstamp, SolveReport* rep) {
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long s = t0; s < H; s += stride) hub_acc[acc_at(s)] = INF;
  for (long long k = t0; k < ncnt; k += stride) cnt[k] = 0ull;
  if (t0 == 0) {
    X[n] = (int)n; Y[n] = (int)n; G[n] = INF;  // dummy vertex n of the padding row
    *done = 0; *ticket = 0u;
    mode[1] = first_mode;
    tstamp[0] = global_ns();
    if (rep) { rep->done = 0; rep->iters = 0; }
  }
}

}  // namespace fsv
