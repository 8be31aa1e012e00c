// C-ABI + host orchestration of the B200 FastSV solver (include/fastsv.h).
//
// Reference hot path: svcc.fastsv_la (/root/reference/pkg/src/svcc/driver.py:64-120)
// and its vertex-level twin svcc.fastsv (algorithms.py:117-167). The kernels
// live in fsv_kernels.cuh; this file owns
//   - the upload pipeline: reference CsrGraph (graph.py:20-52) -> device
//     oriented layout (one entry per undirected edge, head-flagged rows,
//     hub-encoded columns, span table, closed-form f_1),
//   - the solve loop: iteration 1 closed form, then batches of
//     [hook, hubfix, (NCCL allreduce-min), shortcut] queued without host
//     syncs; the host reads one 4-byte convergence flag per batch,
//   - result marshalling into the reference's RunResult/trace shape.
#include "../../include/fastsv.h"
#include "fsv_kernels.cuh"
#include "fsv_variants.cuh"

#include <cub/cub.cuh>
#include <cuda/std/functional>
#include <thrust/iterator/counting_iterator.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <omp.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

using namespace fsv;

// ---------------------------------------------------------------------------
// errors

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(x)                                                                       \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      return fail(FSV_ERR_RUNTIME, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_), \
                  __FILE__, __LINE__, #x);                                                \
  } while (0)

extern "C" const char* fsv_last_error(void) { return g_err.c_str(); }
extern "C" int fsv_abi_version(void) { return FSV_ABI_VERSION; }

extern "C" int fsv_device_count(int* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    if (count) *count = 0;
    return fail(FSV_ERR_RUNTIME, "no CUDA device: %s", cudaGetErrorString(e));
  }
  if (count) *count = c;
  return FSV_OK;
}

// ---------------------------------------------------------------------------
// NCCL, resolved at runtime so the library loads on hosts without NCCL

struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi g_nccl;

static int nccl_load() {
  if (g_nccl.loaded) return FSV_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail(FSV_ERR_RUNTIME, "cannot load NCCL: %s", dlerror());
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.AllReduce || !g_nccl.AllGather || !g_nccl.CommDestroy)
    return fail(FSV_ERR_RUNTIME, "NCCL library lacks required symbols");
  g_nccl.loaded = true;
  return FSV_OK;
}

#define NCCL_TRY(x)                                                                        \
  do {                                                                                     \
    ncclResult_t r_ = (x);                                                                 \
    if (r_ != ncclSuccess)                                                                 \
      return fail(FSV_ERR_RUNTIME, "NCCL error %d (%s) at %s:%d", (int)r_,                \
                  g_nccl.GetErrorString ? g_nccl.GetErrorString(r_) : "?", __FILE__, __LINE__); \
  } while (0)

// ---------------------------------------------------------------------------
// device buffer helper

// Device buffer that only reallocates when it must grow (uploads of
// successive graphs reuse the same memory; cudaFree synchronises the device).
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;    // elements requested by the last alloc
  size_t cap = 0;  // elements allocated
  cudaError_t alloc(size_t count) {
    n = count;
    if (p && count <= cap) return cudaSuccess;
    free();
    n = count;
    cap = std::max<size_t>(count, 1);
    return cudaMalloc(&p, cap * sizeof(T));
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cap = 0;
  }
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { free(); }
};

// hub table + hot accumulators within the 227 KB opt-in shared memory
static constexpr int kHubMax = (SMEM_OPTIN_INTS - HOT_ACC) / 1024 * 1024;
// Default table: 192 KB of shared memory with the hot accumulators. Above
// that the carve-out leaves ~28 KB of L1 and the random global gathers of the
// sweep and the push run at half rate (tools/gather_smem_probe.cu: 139 vs
// 250 G gathers/s); the 8 K least connected hubs are worth less than that
// (config 2: 0.533 -> 0.523 ms, push 42 -> 31 us).
static constexpr int kHubAuto = 192 * 1024 / (int)sizeof(int) - HOT_ACC;
static_assert(kHubAuto <= kHubMax && kHubAuto % 4 == 0, "default hub table size");
// With the L2 rank tier (vectors over L2) the default table is smaller still:
// the freed L1 (~124 KB) caches the most connected tier slots of the compact
// G_hub, which the tier gathers in degree-rank order (config 5: 23.4 ms at
// 47104 slots, 19.8 ms at 24576, 20.0 ms at 16384).
static constexpr int kHubAutoTier = 24576;
static constexpr int kHubMinDegree = 32;  // below this a hub slot buys nothing
static constexpr long long kTierMinN = 1LL << 23;   // rank tier only when the vectors overflow L2
#ifndef FSV_TIER_MIN_DEG
#define FSV_TIER_MIN_DEG 8
#endif
#ifndef FSV_TIER_MAX_M
#define FSV_TIER_MAX_M 4   // config 5: 1 M 17.5 ms, 2 M 15.3, 4 M 14.6, 8 M 14.9, 16 M 15.8 (every slot is refreshed per vertex pass)
#endif
static constexpr int kTierMinDegree = FSV_TIER_MIN_DEG;
static constexpr long long kTierMax = (long long)FSV_TIER_MAX_M << 20;   // 4M: 16 MB of gf + 16 MB of accumulators
#ifndef FSV_SMALL_TASKS
#define FSV_SMALL_TASKS 4
#endif
#ifndef FSV_GRAPH_IF
#define FSV_GRAPH_IF 0
#endif
#ifndef FSV_GRAPH_BODY
#define FSV_GRAPH_BODY 2
#endif
static constexpr int kTraceCap = 4096;    // iteration cap of the counter array
// The minority sweep replaces a dense sweep when the listed vertices' degree
// sum is at most 1/kMinorityDiv of the stored directed entries (it gathers
// from global memory what the dense sweep mostly gathers from shared memory).
#ifndef FSV_MINORITY_DIV
#define FSV_MINORITY_DIV 16
#endif
static constexpr long long kMinorityDiv = FSV_MINORITY_DIV;

struct fsv_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;            // upload: column chunks H2D
  std::vector<cudaEvent_t> chunk_ev;             // one per column chunk
  // graph layout
  bool ready = false;
  int64_t n = 0, m_dir = 0, E = 0, Epad = 0;
  int R = 0, H = 0, HT = 0;   // shared-memory hub slots, all tier slots
  int tiles = 1;               // column-range tiles of the layout (k_tile_pass)
  DBuf<uint32_t> ecol;
  uint32_t* ecolp = nullptr;   // layout start inside ecol
  DBuf<int> span_row, hub_id, f1;
  // full symmetric CSR of this rank's rows, for sparse (push) iterations
  DBuf<int64_t> csr_off;
  DBuf<int> csr_off32;       // int32 copy when the offsets fit (f_1 pass)
  bool off32 = false;
  DBuf<int> csr_cols;
  // the symmetric CSR the solve reads: csr_off/csr_cols, or the caller's
  // device arrays of a borrowed upload (fsv_upload_csr_device)
  const int64_t* offp = nullptr;
  const int* colsp = nullptr;
  int64_t col_base = 0, row_begin = 0, row_end = 0;
  int64_t csr_local = 0;   // entries of this rank's rows in csr_cols
  // changed-gf lists of the vertex pass (one region per warp)
  DBuf<int> dlist, dcount, mode;
  DBuf<PushChunk> chunks;   // long-row chunks of a sparse iteration
  // upload workspace (grow-only, reused across uploads)
  struct {
    DBuf<unsigned long long> bad;
    DBuf<int> deg, ids, deg_sorted, ids_sorted, slot_of, nzflag, nzidx, nzrows;
    DBuf<long long> cnt, out_off, nzoff, carry_e;
    DBuf<int> carry_r;
    DBuf<unsigned char> tmp;
    DBuf<int64_t> cols64;
    DBuf<uint32_t> etmp, etmp2;
    // column-range tiling: runs per row, their bases, sort keys/ids, lengths,
    // rows, sources, segment sizes/offsets
    DBuf<int> t_runs, t_ids, t_len, t_row;
    DBuf<long long> t_base, t_src, t_seg;
    DBuf<uint32_t> t_key;
    DBuf<int4> pieces;
    DBuf<long long> hrow;
    DBuf<unsigned long long> hkept;
    DBuf<int> piece_kept;
  } ws;
  long long rcap = 0;
  int dgrid = 1;
  // solve state
  DBuf<int> xb, gb, G_hub, hub_acc, done;   // xb and f1: parent buffers, gb: gf
  int* hacc = nullptr;   // hub accumulator start inside hub_acc
  int* X = nullptr;
  int* Y = nullptr;
  int* G = nullptr;
  DBuf<unsigned long long> cnt;
  DBuf<unsigned int> ticket;
  DBuf<unsigned> partials;
  int* h_done = nullptr;  // pinned
  // graph mode: the final iteration packs the done flag and the trace of the
  // first STAGE_ITERS iterations into one report; one copy brings it back
  DBuf<SolveReport> rep;
  SolveReport* h_rep = nullptr;   // pinned
  // pageable host transfers: ring of pinned staging buffers (staged_h2d/d2h)
  void* stage_buf[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t stage_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  bool stage_used[4] = {false, false, false, false};
  int stage_next = 0;
  // hooking variants (fsv_variants.cuh): row ids of the stored entries, two
  // extra vectors, and where the labels of the last solve live
  DBuf<int> var_rows, var_t, var_g;
  bool var_rows_ready = false;
  bool variant = false;
  const int* labels_src = nullptr;
  std::vector<cudaEvent_t> events;
  // profile mode: events around every kernel of iteration k: [k][0..7]
  std::vector<cudaEvent_t> pev;
  bool profile = false;
  float hook_ms = 0, hubfix_ms = 0, shortcut_ms = 0, first_ms = 0, allreduce_ms = 0, push_ms = 0;
  int hook_launches = 0;
  int policy = 0;
  double threshold = 0.1;
  int minority = 1;           // fsv_set_minority_sweep
  std::vector<int> h_mode;
  // results of the last solve
  int iterations = 0;
  int components = 0;
  float solve_ms = 0.f;
  std::vector<unsigned long long> h_cnt;
  std::vector<float> iter_ms;
  int labels_ready = 0;
  // device Labeling of the last solve (fsv_get_labeling), built on demand
  bool labeling_ready = false;
  struct {
    DBuf<unsigned> cnt;
    DBuf<int> reps32;
    DBuf<int64_t> reps, sizes, labels;
    DBuf<unsigned char> tmp;
    long long count = 0;
  } lab;
  int host_syncs = 0, launches = 0;
  int hub_limit = kHubAuto;
  bool hub_auto = true;        // default table size (smaller when the rank tier is used)
  long long tile_width = 0;   // fsv_set_tile_width: 0 off, > 0 vertices per column tile, < 0 auto
  // device loop control + CUDA-graph (conditional WHILE) of the iteration loop
  DBuf<int> iterbuf;
  DBuf<unsigned long long> tstamp;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  cudaGraphConditionalHandle graph_cond = 0;
  cudaGraphConditionalHandle graph_cond_next = 0;   // IF node of the body's second iteration
  bool graph_half2 = false;                          // capturing the body's first iteration
  bool graph_dirty = true;
  int graph_key_policy = -1, graph_key_cap = -1;
  double graph_key_thr = -1.0;
  std::vector<long long> graph_key;   // every pointer/size the captured launches use
  bool use_graph = true;
  int sc_grid = 296;  // resident blocks of the vertex-pass kernels
  // multi-GPU
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  bool graph_comm_failed = false;   // NCCL refused capture into the loop body: host loop
  // sparse-iteration delta exchange: this rank's lowered entries (index,
  // value), their count, and the gathered lists of all ranks
  DBuf<int2> dx_list, dx_all;
  DBuf<unsigned> dx_cnt;
  unsigned* h_dx_cnt = nullptr;     // pinned, kGroupMax + 256 entries
  long long xbytes = 0;             // bytes this rank sent over the exchange in the last solve
  int delta_x = 0, dense_x = 0;     // exchanges of each kind in the last solve
};

static int ensure_events(fsv_ctx* c, size_t count) {
  while (c->events.size() < count) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    c->events.push_back(e);
  }
  return FSV_OK;
}

// ---- pageable host transfers ------------------------------------------------
// The drop-in receives plain numpy arrays (pageable memory). A cudaMemcpy
// from pageable memory is staged by the driver through one host thread;
// here host threads copy 8 MB pieces into a ring of pinned buffers while the
// copy engine moves the previous pieces, so the transfer runs near the
// pinned rate. Pinned/registered buffers take the direct path.
constexpr size_t kStageBytes = 8u << 20;
constexpr int kStageBufs = 4;

static bool is_pageable(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

static int stage_init(fsv_ctx* c) {
  for (int i = 0; i < kStageBufs; ++i) {
    if (!c->stage_buf[i]) CUDA_TRY(cudaMallocHost(&c->stage_buf[i], kStageBytes));
    if (!c->stage_ev[i]) CUDA_TRY(cudaEventCreateWithFlags(&c->stage_ev[i], cudaEventDisableTiming));
  }
  return FSV_OK;
}

static void par_memcpy(void* dst, const void* src, size_t bytes) {
  constexpr size_t piece = 512u << 10;
  const long long np = (long long)((bytes + piece - 1) / piece);
  const int T = (int)std::min<long long>(np, std::min(16, omp_get_max_threads()));
  if (T <= 1) {
    memcpy(dst, src, bytes);
    return;
  }
#pragma omp parallel for num_threads(T) schedule(static)
  for (long long i = 0; i < np; ++i) {
    const size_t o = (size_t)i * piece;
    memcpy((char*)dst + o, (const char*)src + o, std::min(piece, bytes - o));
  }
}

// Host (pageable) -> device through the staging ring, ordered on stream s.
static int staged_h2d(fsv_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  int rc = stage_init(c);
  if (rc) return rc;
  for (size_t o = 0; o < bytes; o += kStageBytes) {
    const size_t b = std::min(kStageBytes, bytes - o);
    const int k = c->stage_next;
    c->stage_next = (k + 1) % kStageBufs;
    if (c->stage_used[k]) CUDA_TRY(cudaEventSynchronize(c->stage_ev[k]));
    par_memcpy(c->stage_buf[k], (const char*)src + o, b);
    CUDA_TRY(cudaMemcpyAsync((char*)dst + o, c->stage_buf[k], b, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaEventRecord(c->stage_ev[k], s));
    c->stage_used[k] = true;
  }
  return FSV_OK;
}

// Device -> host (pageable): up to kStageBufs pieces in flight, each copied
// out by the host threads as it lands. Returns when dst holds the data.
static int staged_d2h(fsv_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  int rc = stage_init(c);
  if (rc) return rc;
  const size_t np = (bytes + kStageBytes - 1) / kStageBytes;
  auto issue = [&](size_t i) -> int {
    const size_t o = i * kStageBytes, b = std::min(kStageBytes, bytes - o);
    const int k = (int)(i % kStageBufs);
    // a staged upload may still be reading this buffer on another stream
    if (c->stage_used[k]) CUDA_TRY(cudaEventSynchronize(c->stage_ev[k]));
    c->stage_used[k] = false;
    CUDA_TRY(cudaMemcpyAsync(c->stage_buf[k], (const char*)src + o, b, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaEventRecord(c->stage_ev[k], s));
    return FSV_OK;
  };
  for (size_t i = 0; i < std::min<size_t>(np, kStageBufs); ++i)
    if ((rc = issue(i))) return rc;
  for (size_t i = 0; i < np; ++i) {
    const int k = (int)(i % kStageBufs);
    CUDA_TRY(cudaEventSynchronize(c->stage_ev[k]));
    const size_t o = i * kStageBytes, b = std::min(kStageBytes, bytes - o);
    par_memcpy((char*)dst + o, c->stage_buf[k], b);
    if (i + kStageBufs < np && (rc = issue(i + kStageBufs))) return rc;
  }
  for (int k = 0; k < kStageBufs; ++k) c->stage_used[k] = false;   // ring drained
  return FSV_OK;
}

// Device -> host copy into a caller buffer of any kind (synchronous).
static int copy_out(fsv_ctx* c, void* dst, const void* src, size_t bytes) {
  if (!bytes) return FSV_OK;
  if (bytes >= (1u << 20) && is_pageable(dst)) return staged_d2h(c, dst, src, bytes, c->stream);
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FSV_OK;
}

extern "C" int fsv_create(int device, fsv_ctx** out) {
  if (!out) return fail(FSV_ERR_CONTRACT, "out pointer is NULL");
  *out = nullptr;
  int count = 0;
  int rc = fsv_device_count(&count);
  if (rc) return rc;
  if (device < 0 || device >= count)
    return fail(FSV_ERR_CONTRACT, "device %d out of range (%d devices)", device, count);
  CUDA_TRY(cudaSetDevice(device));
  fsv_ctx* c = new fsv_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMallocHost(&c->h_done, sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&c->h_rep, sizeof(SolveReport)) != cudaSuccess ||
      c->rep.alloc(1) != cudaSuccess) {
    delete c;
    return fail(FSV_ERR_RUNTIME, "stream/pinned allocation failed");
  }
  c->stream = c->own_stream;
  if (cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return fail(FSV_ERR_RUNTIME, "copy stream creation failed");
  }
  {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_shortcut, SC_THREADS, 0);
    c->sc_grid = std::max(1, per_sm) * c->sm_count;
  }
  const int hook_smem = std::max((kHubMax + HOT_ACC) * (int)sizeof(int), PUSH_SCRATCH_BYTES);
  cudaError_t e = cudaSuccess;
  for (const void* fn : {(const void*)k_hook<true, false, STEPS>, (const void*)k_hook<true, true, STEPS>,
                         (const void*)k_hook<true, false, 1>, (const void*)k_hook<true, true, 1>})
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, hook_smem);
  if (e != cudaSuccess) {
    delete c;
    return fail(FSV_ERR_RUNTIME, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  *out = c;
  return FSV_OK;
}

extern "C" int fsv_destroy(fsv_ctx* c) {
  if (!c) return FSV_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto e : c->events) cudaEventDestroy(e);
  for (auto e : c->pev) cudaEventDestroy(e);
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  if (c->graph) cudaGraphDestroy(c->graph);
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  if (c->h_done) cudaFreeHost(c->h_done);
  if (c->h_rep) cudaFreeHost(c->h_rep);
  if (c->h_dx_cnt) cudaFreeHost(c->h_dx_cnt);
  for (int i = 0; i < 4; ++i) {
    if (c->stage_buf[i]) cudaFreeHost(c->stage_buf[i]);
    if (c->stage_ev[i]) cudaEventDestroy(c->stage_ev[i]);
  }
  for (auto e : c->chunk_ev) cudaEventDestroy(e);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
  return FSV_OK;
}

extern "C" int fsv_set_stream(fsv_ctx* c, void* s) {
  if (!c) return fail(FSV_ERR_CONTRACT, "NULL context");
  c->stream = s ? (cudaStream_t)s : c->own_stream;
  return FSV_OK;
}

// ---------------------------------------------------------------------------
// upload pipeline kernels

// degrees + ids for the sort, and the offsets sanity check (non-decreasing)
constexpr uint32_t DROP = 0xffffffffu;
#ifndef FSV_HUGE_ROW
#define FSV_HUGE_ROW 512
#endif
#ifndef FSV_PIECE
#define FSV_PIECE 1024
#endif
#ifndef FSV_LONG_ROW
#define FSV_LONG_ROW 32          // rows longer than this are encoded/compacted by a whole warp
#endif
constexpr long long HUGE_ROW = FSV_HUGE_ROW;  // rows longer than this are cut into pieces
constexpr long long PIECE = FSV_PIECE;        // entries per piece

// Also lists the pieces of this rank's rows longer than HUGE_ROW (what
// k_find_huge does, in the same pass over the offsets). The offsets are not
// validated yet here, so the list is bounded (ctr[2] flags an overflow) and
// the upload fails on the non-decreasing check before anything reads it.
__global__ void k_degree(const int64_t* __restrict__ off, long long n, int* __restrict__ deg,
                         int* __restrict__ ids, unsigned long long* bad, long long row_begin, long long row_end,
                         long long* __restrict__ hrow, int4* __restrict__ pieces, unsigned long long* ctr,
                         long long max_huge, long long max_pieces) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n;
       u += (long long)gridDim.x * blockDim.x) {
    const int64_t d = off[u + 1] - off[u];
    if (d < 0) atomicMin(bad, (unsigned long long)u);
    deg[u] = (int)d;
    ids[u] = (int)u;
    if (d > HUGE_ROW && u >= row_begin && u < row_end) {
      const long long np = (d + PIECE - 1) / PIECE;
      const unsigned long long h = atomicAdd(ctr, 1ull);
      const unsigned long long b = atomicAdd(ctr + 1, (unsigned long long)np);
      if ((long long)h >= max_huge || (long long)(b + np) > max_pieces) {
        ctr[2] = 1ull;
        continue;
      }
      hrow[h] = u - row_begin;
      for (long long j = 0; j < np; ++j) pieces[b + j] = make_int4((int)u, (int)j, (int)j + 1, (int)h);
    }
  }
}

// pos[v] = position of v in the degree-descending order (ties by id); hubs
// are the first H positions, so a vertex's hub slot is its position.
__global__ void k_positions(const int* __restrict__ sorted_ids, long long n, int H,
                            int* __restrict__ pos, int* __restrict__ hub_id) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int v = sorted_ids[i];
    pos[v] = (int)i;
    if (i < H) hub_id[i] = v;
  }
}

// number of leading entries >= thr in a descending array (one warp, binary search)
__global__ void k_count_ge(const int* __restrict__ sorted_desc, long long n, int thr, long long* out) {
  if (threadIdx.x != 0) return;
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (sorted_desc[mid] >= thr) lo = mid + 1; else hi = mid;
  }
  *out = lo;
}


__device__ __forceinline__ uint32_t encode_col(int v, int pv, int H) {
  return pv < H ? (HUB | (uint32_t)pv) : (uint32_t)v;
}

// Orientation pass 1: the edge {u, v} is kept once, in the row of the
// endpoint that comes later in the degree order (so columns point at
// high-degree vertices). Each entry gathers pos[v] once and is written,
// encoded, at its own position in `tmp` (DROP if not kept); per-row kept
// counts (+1 header) go to cnt. Warp = 32 consecutive rows: short rows one
// per lane, long rows by the whole warp. Also range-checks the columns.
template <typename ColT>
__global__ void k_orient_encode(const int64_t* __restrict__ off, const ColT* __restrict__ cols,
                                long long col_base, long long row_begin, long long rows, long long n,
                                const int* __restrict__ pos, int H, uint32_t* __restrict__ tmp,
                                long long* __restrict__ cnt, int* __restrict__ nzflag,
                                unsigned long long* bad) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long w0 = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; w0 < rows;
       w0 += nw * 32) {
    const long long r = w0 + lane;
    long long lo = 0, hi = 0;
    int pu = 0;
    if (r < rows) {
      const long long u = row_begin + r;
      lo = off[u] - col_base;
      hi = off[u + 1] - col_base;
      pu = pos[u];
    }
    const bool huge = hi - lo > HUGE_ROW;        // cut into pieces (k_piece_encode)
    if (huge) hi = lo;
    const bool is_long = hi - lo > FSV_LONG_ROW;
    long long k = 0;
    if (!is_long) {
      // 4 entries of the lane's row in flight (column loads, then pos gathers)
      for (long long e = lo; e < hi; e += 4) {
        long long v[4];
        int pv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = e + q < hi ? (long long)cols[e + q] : 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) pv[q] = (e + q < hi && v[q] >= 0 && v[q] < n) ? pos[v[q]] : INF;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (e + q >= hi) break;
          uint32_t code = DROP;
          if (v[q] < 0 || v[q] >= n) {
            atomicMin(bad, (unsigned long long)(e + q));
          } else if (pv[q] < pu) {
            code = encode_col((int)v[q], pv[q], H);
            ++k;
          }
          tmp[e + q] = code;
        }
      }
    }
    unsigned lm = __ballot_sync(0xffffffffu, is_long);
    while (lm) {
      const int src = __ffs(lm) - 1;
      lm &= lm - 1;
      const long long slo = __shfl_sync(0xffffffffu, lo, src);
      const long long shi = __shfl_sync(0xffffffffu, hi, src);
      const int spu = __shfl_sync(0xffffffffu, pu, src);
      long long sk = 0;
      // 8 entries per lane in flight (column loads, then pos gathers)
      for (long long e0 = slo; e0 < shi; e0 += 8 * 32) {
        long long v[8];
        int pv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const long long e = e0 + lane + 32 * j;
          v[j] = e < shi ? (long long)cols[e] : -2;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) pv[j] = (v[j] >= 0 && v[j] < n) ? pos[v[j]] : INF;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const long long e = e0 + lane + 32 * j;
          if (e >= shi) continue;
          uint32_t code = DROP;
          if (v[j] < 0 || v[j] >= n) atomicMin(bad, (unsigned long long)e);
          else if (pv[j] < spu) { code = encode_col((int)v[j], pv[j], H); ++sk; }
          tmp[e] = code;
        }
      }
      for (int o = 16; o; o >>= 1) sk += __shfl_xor_sync(0xffffffffu, sk, o);
      if (lane == src) k = sk;
    }
    if (r < rows && !huge) {
      cnt[r] = k ? k + 1 : 0;  // + header entry
      nzflag[r] = k > 0;
    }
  }
}

// Pieces of rows longer than HUGE_ROW: one warp per piece (listed by the
// host), 8 entries per lane in flight; kept counts summed per row.
template <typename ColT>
__global__ void k_piece_encode(const int4* __restrict__ pieces, const unsigned long long* npieces_p,
                               long long u0, long long u1, const int64_t* __restrict__ off,
                               const ColT* __restrict__ cols, long long col_base, long long n,
                               const int* __restrict__ pos, int H, uint32_t* __restrict__ tmp,
                               unsigned long long* __restrict__ row_kept, int* __restrict__ piece_kept,
                               unsigned long long* bad) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  const long long npieces = (long long)*npieces_p;
  for (long long q = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < npieces; q += nw) {
    const int4 pc = pieces[q];                      // (row u, piece start, piece end, huge-row index)
    const int u = pc.x;
    if (u < u0 || u >= u1) continue;                // another chunk's row
    const long long base = off[u] - col_base;
    const long long lo = base + (long long)pc.y * PIECE, hi = min(base + (long long)pc.z * PIECE,
                                                                  off[u + 1] - col_base);
    const int pu = pos[u];
    unsigned long long k = 0;
    for (long long e0 = lo; e0 < hi; e0 += 8 * 32) {
      long long v[8];
      int pv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const long long e = e0 + lane + 32 * j;
        v[j] = e < hi ? (long long)cols[e] : -2;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) pv[j] = (v[j] >= 0 && v[j] < n) ? pos[v[j]] : INF;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const long long e = e0 + lane + 32 * j;
        if (e >= hi) continue;
        uint32_t code = DROP;
        if (v[j] < 0 || v[j] >= n) atomicMin(bad, (unsigned long long)e);
        else if (pv[j] < pu) { code = encode_col((int)v[j], pv[j], H); ++k; }
        tmp[e] = code;
      }
    }
    for (int o = 16; o; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    if (lane == 0) {
      piece_kept[q] = (int)k;
      if (k) atomicAdd(row_kept + pc.w, k);
    }
  }
}

// Huge rows: per-row counts from the pieces (+ header), and the output
// cursor for k_piece_compact; `hrow[i]` = (row - row_begin) of huge row i.
__global__ void k_huge_rows(const long long* __restrict__ hrow, const unsigned long long* nh_p,
                            long long r0, long long r1, const unsigned long long* row_kept,
                            long long* __restrict__ cnt, int* __restrict__ nzflag) {
  const long long nh = (long long)*nh_p;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nh;
       i += (long long)gridDim.x * blockDim.x) {
    if (hrow[i] < r0 || hrow[i] >= r1) continue;
    const long long k = (long long)row_kept[i];
    cnt[hrow[i]] = k ? k + 1 : 0;
    nzflag[hrow[i]] = k > 0;
  }
}

// Pieces of a huge row are consecutive in the piece list (piece j of the
// row at index q has its predecessors at q-j .. q-1), so each piece's output
// offset is the row offset plus its predecessors' kept counts: the row keeps
// its column order, deterministically.
__global__ void k_piece_compact(const int4* __restrict__ pieces, const unsigned long long* npieces_p,
                                long long u0, long long u1, const int64_t* __restrict__ off,
                                long long col_base, const uint32_t* __restrict__ tmp,
                                const long long* __restrict__ hrow, const long long* __restrict__ out_off,
                                const int* __restrict__ piece_kept, uint32_t* __restrict__ ecol) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  const long long npieces = (long long)*npieces_p;
  for (long long q = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < npieces; q += nw) {
    const int4 pc = pieces[q];
    const int u = pc.x;
    if (u < u0 || u >= u1) continue;
    const long long base = off[u] - col_base;
    const long long lo = base + (long long)pc.y * PIECE, hi = min(base + (long long)pc.z * PIECE,
                                                                  off[u + 1] - col_base);
    long long before = 0;
    for (long long i = q - pc.y + lane; i < q; i += 32) before += piece_kept[i];
    for (int o = 16; o; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
    long long o = out_off[hrow[pc.w]] + 1 + before;
    for (long long e0 = lo; e0 < hi; e0 += 8 * 32) {
      uint32_t code[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const long long e = e0 + lane + 32 * j;
        code[j] = e < hi ? tmp[e] : DROP;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bool keep = code[j] != DROP;
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        if (keep) ecol[o + __popc(b & ((1u << lane) - 1u))] = code[j];
        o += __popc(b);
      }
    }
  }
}

// Column-range tiling of a built layout (fsv_set_tile_width). Every row
// segment (header + kept codes, ecol) is cut into runs of consecutive codes
// in the same column tile (hub-coded columns, gathered from shared memory or
// the L2 tier rather than from G, count as tile 0); the runs are stably
// sorted by tile and written back, each behind its own copy of the row's
// header: all rows' tile-0 runs, then tile 1's, ... The dense sweep then
// gathers gf from, and reduces into, one W-vertex slice of the vertex
// vectors at a time, which stays L2-resident. A row split over runs emits
// one partial row minimum per run (min-reductions are idempotent).
__device__ __forceinline__ uint32_t code_tile(uint32_t c, long long w) {
  return (c & HUB) ? 0u : (uint32_t)((long long)c / w);
}

// Runs per row segment i = [nzoff[i] + 1, nzoff[i + 1]) (the last ends at E).
template <bool EMIT>
__global__ void k_tile_runs(const uint32_t* __restrict__ ecol, const long long* __restrict__ nzoff,
                            const int* __restrict__ nzrows, long long R, long long E, long long w,
                            int* __restrict__ runs, const long long* __restrict__ run_base,
                            uint32_t* __restrict__ key, long long* __restrict__ src, int* __restrict__ len,
                            int* __restrict__ row) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < R; i += (long long)gridDim.x * blockDim.x) {
    const long long lo = nzoff[i] + 1, hi = (i + 1 < R) ? nzoff[i + 1] : E;
    long long k = EMIT ? run_base[i] : 0;
    int cnt = 0;
    uint32_t cur = 0xffffffffu;
    long long start = lo;
    for (long long e = lo; e < hi; ++e) {
      const uint32_t t = code_tile(ecol[e], w);
      if (t != cur) {
        if (EMIT && cnt) { key[k] = cur; src[k] = start; len[k] = (int)(e - start); row[k] = nzrows[i]; ++k; }
        cur = t;
        start = e;
        ++cnt;
      }
    }
    if (EMIT) {
      if (cnt) { key[k] = cur; src[k] = start; len[k] = (int)(hi - start); row[k] = nzrows[i]; }
    } else {
      runs[i] = cnt;
    }
  }
}

__global__ void k_iota(int* __restrict__ a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    a[i] = (int)i;
}

__global__ void k_tile_lens(const int* __restrict__ ids, const int* __restrict__ len, long long M,
                            long long* __restrict__ seg) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < M; k += (long long)gridDim.x * blockDim.x)
    seg[k] = len[ids[k]] + 1;
}

// Sorted run k: header at out[k], its codes behind it; the span table's
// segment arrays (nzrows, nzoff) follow the new order. A thread per run
// (runs are short: at most a row), its dependent loads independent of the
// other threads'; runs over 32 codes are copied by the whole warp.
__global__ void k_tile_scatter(const uint32_t* __restrict__ ecol, const int* __restrict__ ids,
                               const long long* __restrict__ src, const int* __restrict__ len,
                               const int* __restrict__ row, const long long* __restrict__ out, long long M,
                               uint32_t* __restrict__ ecol2, int* __restrict__ nzrows, long long* __restrict__ nzoff) {
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < M; base += stride) {   // block-uniform
    const long long k = base + threadIdx.x;
    long long o = 0, s0 = 0;
    int l = 0;
    if (k < M) {
      const int id = ids[k];
      o = out[k];
      s0 = src[id];
      l = len[id];
      const int u = row[id];
      ecol2[o] = HDR | (uint32_t)u;
      nzrows[k] = u;
      nzoff[k] = o;
      if (l <= 32)
        for (int j = 0; j < l; ++j) ecol2[o + 1 + j] = ecol[s0 + j];
    }
    unsigned lm = __ballot_sync(0xffffffffu, l > 32);
    while (lm) {
      const int q = __ffs(lm) - 1;
      lm &= lm - 1;
      const long long qo = __shfl_sync(0xffffffffu, o, q), qs = __shfl_sync(0xffffffffu, s0, q);
      const int ql = __shfl_sync(0xffffffffu, l, q);
      for (int j = lane; j < ql; j += 32) ecol2[qo + 1 + j] = ecol[qs + j];
    }
  }
}

// Orientation pass 2 (no gathers): header + kept entries of each row, in
// order, at out_off[r]; nzrows/nzoff for the span table.
__global__ void k_orient_compact(const int64_t* __restrict__ off, long long col_base, long long row_begin,
                                 long long rows, const uint32_t* __restrict__ tmp,
                                 const long long* __restrict__ out_off, const int* __restrict__ nzidx,
                                 uint32_t* __restrict__ ecol, int* __restrict__ nzrows,
                                 long long* __restrict__ nzoff) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long w0 = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; w0 < rows;
       w0 += nw * 32) {
    const long long r = w0 + lane;
    long long lo = 0, hi = 0, o0 = 0;
    bool has = false;
    if (r < rows) {
      const long long u = row_begin + r;
      lo = off[u] - col_base;
      hi = off[u + 1] - col_base;
      o0 = out_off[r];
      has = out_off[r + 1] > o0;
      if (has) {
        ecol[o0] = HDR | (uint32_t)u;
        const int z = nzidx[r];
        nzrows[z] = (int)u;
        nzoff[z] = o0;
      }
    }
    if (hi - lo > HUGE_ROW) hi = lo;     // entries placed by k_piece_compact
    const bool is_long = has && hi - lo > FSV_LONG_ROW;
    if (has && !is_long) {
      long long o = o0 + 1;
      for (long long e = lo; e < hi; e += 4) {
        uint32_t code[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) code[q] = e + q < hi ? tmp[e + q] : DROP;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (code[q] != DROP) ecol[o++] = code[q];
      }
    }
    unsigned lm = __ballot_sync(0xffffffffu, is_long);
    while (lm) {
      const int src = __ffs(lm) - 1;
      lm &= lm - 1;
      const long long slo = __shfl_sync(0xffffffffu, lo, src);
      const long long shi = __shfl_sync(0xffffffffu, hi, src);
      long long o = __shfl_sync(0xffffffffu, o0, src) + 1;
      for (long long e0 = slo; e0 < shi; e0 += 8 * 32) {
        uint32_t code[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const long long e = e0 + lane + 32 * j;
          code[j] = e < shi ? tmp[e] : DROP;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const bool keep = code[j] != DROP;
          const unsigned b = __ballot_sync(0xffffffffu, keep);
          if (keep) ecol[o + __popc(b & ((1u << lane) - 1u))] = code[j];
          o += __popc(b);
        }
      }
    }
  }
}

// Chains the per-chunk scans: after chunk k's exclusive scans of rows
// [r0, r1) (seeded with carry[k]), the totals up to r1 become carry[k+1]
// and the out_off/nzidx entries at r1 (read by the compaction of chunk k).
__global__ void k_chunk_carry(const long long* __restrict__ cnt, const int* __restrict__ nzflag,
                              long long* __restrict__ out_off, int* __restrict__ nzidx, long long r0,
                              long long r1, long long* carry_e, int* carry_r, int k) {
  long long e = carry_e[k];
  int z = carry_r[k];
  if (r1 > r0) {
    e = out_off[r1 - 1] + cnt[r1 - 1];
    z = nzidx[r1 - 1] + nzflag[r1 - 1];
  }
  carry_e[k + 1] = e;
  carry_r[k + 1] = z;
  out_off[r1] = e;
  nzidx[r1] = z;
}

__global__ void k_pad(uint32_t* ecol, long long E, long long Epad, int n, int* nzrows, int R,
                      long long* nzoff) {
  for (long long e = E + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < Epad;
       e += (long long)gridDim.x * blockDim.x)
    ecol[e] = HDR | (uint32_t)n;  // empty rows of the dummy vertex n (gf = INF)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    nzrows[R] = n;
    nzoff[R] = E;
  }
}

// span_row[s] = vertex of the row whose entries include s*task when that
// entry is an edge (the row started in an earlier span), else -1.
__global__ void k_span_row(const long long* __restrict__ nzoff, const int* __restrict__ nzrows,
                           int R1, long long nspans, int task, int* __restrict__ span_row) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < nspans;
       s += (long long)gridDim.x * blockDim.x) {
    const long long target = s * task;
    int lo = 0, hi = R1;  // upper_bound over nzoff[0..R1)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (nzoff[mid] <= target) lo = mid + 1; else hi = mid;
    }
    const int r = lo - 1;
    span_row[s] = (r < 0 || nzoff[r] == target) ? -1 : nzrows[r];
  }
}

// f_1[u] = min(u, first (= smallest) column of row u) for rows this rank owns;
// other rows get `outside` (INF before an allreduce-min assembles the global
// vector, or u itself when there is no communicator).
template <typename ColT>
__global__ void k_f1(const int64_t* __restrict__ off, const ColT* __restrict__ cols,  // (ColT = int)
                     long long col_base, long long row_begin, long long row_end, long long n,
                     int* __restrict__ f1, bool outside_inf) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n;
       u += (long long)gridDim.x * blockDim.x) {
    int val = outside_inf ? INF : (int)u;
    if (u >= row_begin && u < row_end) {
      val = (int)u;
      if (off[u + 1] > off[u]) val = min(val, (int)cols[off[u] - col_base]);
    }
    f1[u] = val;
  }
}

// In-solve f_1 for the full single-rank row range: 4 vertices per thread,
// offsets as two 16-byte loads, the four first-column loads in flight together.
template <typename OffT>
__global__ void k_f1_solve(const OffT* __restrict__ off, const int* __restrict__ cols, long long n,
                           int* __restrict__ f1) {
  const long long n4 = n >> 2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= n4;
       i += (long long)gridDim.x * blockDim.x) {
    const long long u0 = i << 2;
    if (u0 + 4 <= n) {
      long long o[5];
      if constexpr (sizeof(OffT) == 4) {
        const int4 a = *reinterpret_cast<const int4*>(off + u0);            // off[u0 .. u0+3]
        o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
      } else {
        const longlong2 a = *reinterpret_cast<const longlong2*>(off + u0);  // off[u0], off[u0+1]
        const longlong2 b = *reinterpret_cast<const longlong2*>(off + u0 + 2);
        o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
      }
      o[4] = off[u0 + 4];
      int4 r;
      int* rp = reinterpret_cast<int*>(&r);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = o[j + 1] > o[j] ? __ldg(cols + o[j]) : INF;
        rp[j] = min((int)(u0 + j), c);
      }
      *reinterpret_cast<int4*>(f1 + u0) = r;
    } else {
      for (long long u = u0; u < n; ++u)
        f1[u] = off[u + 1] > off[u] ? min((int)u, cols[off[u]]) : (int)u;
    }
  }
}

// rows no rank owned stay isolated (never index with INF)
__global__ void k_f1_fix(int* __restrict__ f1, long long n) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n;
       u += (long long)gridDim.x * blockDim.x)
    if (f1[u] == INF) f1[u] = (int)u;
}

__global__ void k_narrow(const int64_t* __restrict__ in, long long m, int* __restrict__ out) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = (int)in[e];
}

// ---- CSR build from an edge list on the device (graph.py:55-97) -------------
// Directed entry (u, v) -> key u << b | v (b id bits, n <= 2^b). A dropped
// pair (self-loop, or out of range: reported) gets the all-ones 2b-bit key,
// which no kept entry has (it would need u == v) and which sorts last.
template <typename IdT>
struct PairT;
template <>
struct PairT<int32_t> { using V = int2; };
template <>
struct PairT<int64_t> { using V = longlong2; };

template <typename IdT>
__global__ void k_edge_keys(const IdT* __restrict__ pairs, long long i0, long long i1, long long n, int b,
                            unsigned long long* __restrict__ keys, unsigned long long* bad) {
  const unsigned long long sent = (1ull << (2 * b)) - 1ull;
  const auto* P = reinterpret_cast<const typename PairT<IdT>::V*>(pairs);
  for (long long i = i0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < i1;
       i += (long long)gridDim.x * blockDim.x) {
    const auto p = P[i];
    const long long u = (long long)p.x, v = (long long)p.y;
    ulonglong2 k = make_ulonglong2(sent, sent);
    if (u < 0 || u >= n || v < 0 || v >= n) {
      atomicMin(bad, (unsigned long long)i);
    } else if (u != v) {
      k.x = ((unsigned long long)u << b) | (unsigned long long)v;
      k.y = ((unsigned long long)v << b) | (unsigned long long)u;
    }
    reinterpret_cast<ulonglong2*>(keys)[i] = k;
  }
}

// Unique-key count without the sentinel: out[0] = entries of the CSR.
__global__ void k_key_count(const unsigned long long* keys, const long long* nuniq, int b, long long* out) {
  const unsigned long long sent = (1ull << (2 * b)) - 1ull;
  const long long u = *nuniq;
  out[0] = (u > 0 && keys[u - 1] == sent) ? u - 1 : u;
}

// CSR from sorted unique keys: cols[i] = v, row_offsets[r] = first entry of
// row >= r (each entry fills the offsets of the rows up to its own when it
// starts a row; the last entry fills the tail).
__global__ void k_csr_from_keys(const unsigned long long* __restrict__ keys, const long long* M_p, long long n,
                                int b, int64_t* __restrict__ off, int* __restrict__ cols) {
  const long long M = *M_p;
  const unsigned long long mask = (1ull << b) - 1ull;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (M == 0) {
    for (long long r = t0; r <= n; r += stride) off[r] = 0;
    return;
  }
  for (long long i = t0; i < M; i += stride) {
    const unsigned long long k = keys[i];
    const long long u = (long long)(k >> b);
    cols[i] = (int)(k & mask);
    const long long up = i ? (long long)(keys[i - 1] >> b) : -1;
    for (long long r = up + 1; r <= u; ++r) off[r] = i;
    if (i == M - 1)
      for (long long r = u + 1; r <= n; ++r) off[r] = M;
  }
}

// A layout with fewer STEP-entry steps than FSV_SMALL_TASKS x the resident
// hook warps is processed one step per warp task (every warp busy) instead
// of STEPS-step tasks (a few long tasks).
static bool small_layout(const fsv_ctx* c, long long Epad) {
  return Epad / STEP < (long long)FSV_SMALL_TASKS * c->sm_count * (HOOK_THREADS / 32);
}

static int grid_for(fsv_ctx* c, long long work, int threads, int per_sm = 8) {
  long long g = (work + threads - 1) / threads;
  g = std::min<long long>(g, (long long)c->sm_count * per_sm);
  return (int)std::max<long long>(g, 1);
}

template <typename ColT>
static DBuf<ColT>& cols_buffer(fsv_ctx* c);
template <>
DBuf<int32_t>& cols_buffer<int32_t>(fsv_ctx* c) { return c->csr_cols; }
template <>
DBuf<int64_t>& cols_buffer<int64_t>(fsv_ctx* c) { return c->ws.cols64; }

// Row offsets of an upload as the host sees them: the full host array, or
// (h == nullptr) device-resident offsets of which the host only fetched the
// entries at 0, row_begin, row_end and n.
struct HostOff {
  const int64_t* h = nullptr;
  int64_t idx[4] = {-1, -1, -1, -1}, val[4] = {0, 0, 0, 0};
  int64_t operator[](int64_t i) const {
    if (h) return h[i];
    for (int k = 0; k < 4; ++k)
      if (idx[k] == i) return val[k];
    return -1;
  }
};

// Offsets come from host h_off (copied up), or, when h_off is NULL, from the
// device array d_off_src (fsv_upload_edges: the context's own csr_off;
// fsv_upload_csr_device: the caller's). Columns come from host h_cols
// (copied up in chunks) or from the device array d_src, indexed by global
// entry (d_src_slice = false: every row's columns, fsv_upload_edges) or by
// entry within this rank's rows (d_src_slice = true). borrow = true uses the
// caller's device arrays in place for the context's lifetime (no copy).
template <typename ColT>
static int upload_impl(fsv_ctx* c, int64_t n, const int64_t* h_off_arr, const ColT* h_cols,
                       int64_t row_begin, int64_t row_end, const ColT* d_src = nullptr,
                       const int64_t* d_off_src = nullptr, bool d_src_slice = false, bool borrow = false) {
  if (!c) return fail(FSV_ERR_CONTRACT, "NULL context");
  if (n < 0) return fail(FSV_ERR_INPUT, "vertex count must be non-negative, got %lld", (long long)n);
  if (n >= (int64_t)IDMASK) return fail(FSV_ERR_INPUT, "n=%lld exceeds the device id range", (long long)n);
  if (!h_off_arr && !d_off_src) return fail(FSV_ERR_CONTRACT, "row_offsets is NULL");
  if (row_begin < 0 || row_end < row_begin || row_end > n)
    return fail(FSV_ERR_CONTRACT, "row range [%lld, %lld) invalid for n=%lld", (long long)row_begin,
                (long long)row_end, (long long)n);
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  HostOff h_off;
  h_off.h = h_off_arr;
  if (!h_off_arr) {
    const int64_t ix[4] = {0, row_begin, row_end, n};
    for (int k = 0; k < 4; ++k) {
      h_off.idx[k] = ix[k];
      CUDA_TRY(cudaMemcpyAsync(&h_off.val[k], d_off_src + ix[k], sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    }
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (h_off[0] != 0) return fail(FSV_ERR_INPUT, "row_offsets[0] must be 0");
  if (h_off[n] < h_off[0]) return fail(FSV_ERR_INPUT, "row_offsets must be non-decreasing");
  const int64_t e_begin = h_off[row_begin], e_end = h_off[row_end];
  const int64_t mloc = e_end - e_begin;
  if (mloc < 0 || e_begin < 0 || e_end > h_off[n]) return fail(FSV_ERR_INPUT, "row_offsets must be non-decreasing");
  if (mloc > 0 && !h_cols && !d_src) return fail(FSV_ERR_CONTRACT, "col_indices is NULL");
  if (borrow && (!d_src || !d_src_slice || !d_off_src || h_off_arr))
    return fail(FSV_ERR_CONTRACT, "borrowed uploads take device offsets and a device column slice");
  // the device column source indexed by global entry
  const ColT* d_src_g = d_src ? (d_src_slice ? d_src - e_begin : d_src) : nullptr;
  c->ready = false;
  c->labels_ready = 0;
  c->labeling_ready = false;
  c->graph_dirty = true;

  const long long rows = row_end - row_begin;
  const bool udbg = getenv("FSV_UPLOAD_DEBUG") != nullptr;
  cudaEvent_t uev[8];
  if (udbg) for (auto& e : uev) cudaEventCreate(&e);
  auto umark = [&](int i) { if (udbg) cudaEventRecord(uev[i], st); };
  umark(0);
  std::vector<cudaEvent_t> dbg_copy_ev, dbg_enc_ev;
  DBuf<int64_t>& d_off = c->csr_off;
  DBuf<ColT>& d_cols = cols_buffer<ColT>(c);
  // offp/colp: the offsets and this rank's columns the layout build reads
  const int64_t* offp = nullptr;
  const ColT* colp = nullptr;
  if (borrow) {
    offp = d_off_src;
    colp = d_src;
  } else {
    if (d_off_src != d_off.p || !d_off.p) CUDA_TRY(d_off.alloc((size_t)n + 1));
    CUDA_TRY(d_cols.alloc((size_t)mloc));
    if (h_off_arr && is_pageable(h_off_arr)) {
      int rc = staged_h2d(c, d_off.p, h_off_arr, sizeof(int64_t) * (n + 1), st);
      if (rc) return rc;
    } else if (h_off_arr) {
      CUDA_TRY(cudaMemcpyAsync(d_off.p, h_off_arr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st));
    }
    else if (d_off_src != d_off.p)
      CUDA_TRY(cudaMemcpyAsync(d_off.p, d_off_src, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, st));
    offp = d_off.p;
    colp = d_cols.p;
  }
  // columns go up in row-aligned chunks on the copy stream, so the degree
  // sort and the orientation of earlier chunks overlap the transfer
  const bool cols_pageable = h_cols && !d_src && mloc > 0 && is_pageable(h_cols);
  std::vector<int64_t> chunk_rows;  // row boundaries, chunk k = [chunk_rows[k], chunk_rows[k+1])
  {
    // eighths of the entries, the last eighth cut geometrically (1/16, 1/32,
    // 1/64, 1/64) so the work trailing the final copy is small
    std::vector<int64_t> cut;  // chunk ends in 1/64ths of mloc
    if (mloc >= ((int64_t)1 << 24) && !d_src && h_off.h) cut = {8, 16, 24, 32, 40, 48, 56, 60, 62, 63, 64};
    else cut = {64};
    if (const char* env = d_src ? nullptr : getenv("FSV_UPLOAD_CHUNKS")) {   // dev: K equal chunks
      const int k_eq = std::max(1, std::min(64, atoi(env)));
      cut.clear();
      for (int k = 1; k <= k_eq; ++k) cut.push_back(64 * k / k_eq);
    }
    const int K = (int)cut.size();
    chunk_rows.push_back(row_begin);
    for (int k = 0; k + 1 < K; ++k) {
      const int64_t target = e_begin + (int64_t)((__int128)mloc * cut[k] / 64);
      int64_t r = std::lower_bound(h_off.h + row_begin, h_off.h + row_end, target) - h_off.h;   // K > 1: host offsets
      r = std::max<int64_t>(r, chunk_rows.back());
      chunk_rows.push_back(std::min<int64_t>(r, row_end));
    }
    chunk_rows.push_back(row_end);
    while (c->chunk_ev.size() < (size_t)K) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->chunk_ev.push_back(e);
    }
    cudaEvent_t off_ready = c->chunk_ev[0];
    CUDA_TRY(cudaEventRecord(off_ready, st));              // d_off allocation/reuse ordering
    CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, off_ready, 0));
    // pageable host columns: staged pieces issued chunk by chunk inside the
    // orientation loop below (the host copies chunk k+1 while the device
    // orients chunk k); pinned ones all go up now
    for (int k = 0; k < K && !cols_pageable; ++k) {
      const int64_t lo = h_off[chunk_rows[k]] - e_begin, hi = h_off[chunk_rows[k + 1]] - e_begin;
      // only non-decreasing offsets are accepted (checked on the device
      // below); until then no copy may leave [0, mloc)
      if (lo < 0 || hi > mloc || (hi < lo && !d_src)) {
        cudaStreamSynchronize(c->copy_stream);
        return fail(FSV_ERR_INPUT, "row_offsets must be non-decreasing");
      }
      if (hi > lo && !d_src)
        CUDA_TRY(cudaMemcpyAsync(d_cols.p + lo, h_cols + lo, sizeof(ColT) * (hi - lo),
                                 cudaMemcpyHostToDevice, c->copy_stream));
      else if (hi > lo && !borrow && d_src_g + e_begin + lo != d_cols.p + lo)   // this rank's slice of a device CSR
        CUDA_TRY(cudaMemcpyAsync(d_cols.p + lo, d_src_g + e_begin + lo, sizeof(ColT) * (hi - lo),
                                 cudaMemcpyDeviceToDevice, c->copy_stream));
      CUDA_TRY(cudaEventRecord(c->chunk_ev[k], c->copy_stream));
      if (udbg) {
        cudaEvent_t e; cudaEventCreate(&e); cudaEventRecord(e, c->copy_stream);
        dbg_copy_ev.push_back(e);
      }
    }
  }
  // rows longer than HUGE_ROW are cut into PIECE-entry pieces so no single
  // warp walks a whole hub row; the list is built on the device from the
  // offsets (which arrive first), counts stay on the device
  const long long max_huge = mloc / HUGE_ROW + 1;
  const long long max_pieces = mloc / PIECE + max_huge + 1;
  CUDA_TRY(c->ws.pieces.alloc((size_t)max_pieces));
  CUDA_TRY(c->ws.hrow.alloc((size_t)max_huge));
  CUDA_TRY(c->ws.hkept.alloc((size_t)max_huge + 3));   // [0..max_huge) kept, then 3 counters
  CUDA_TRY(c->ws.piece_kept.alloc((size_t)max_pieces));
  CUDA_TRY(cudaMemsetAsync(c->ws.hkept.p, 0, sizeof(unsigned long long) * (max_huge + 3), st));
  unsigned long long* huge_ctr = c->ws.hkept.p + max_huge;      // [0] huge rows, [1] pieces, [2] overflow

  // degrees (+ offsets check), stable degree order, positions, hubs
  DBuf<unsigned long long>& d_bad = c->ws.bad;
  CUDA_TRY(d_bad.alloc(2));
  CUDA_TRY(cudaMemsetAsync(d_bad.p, 0xff, 2 * sizeof(unsigned long long), st));
  auto& deg = c->ws.deg;
  auto& ids = c->ws.ids;
  auto& deg_sorted = c->ws.deg_sorted;
  auto& ids_sorted = c->ws.ids_sorted;
  auto& pos = c->ws.slot_of;
  CUDA_TRY(deg.alloc(n)); CUDA_TRY(ids.alloc(n));
  CUDA_TRY(deg_sorted.alloc(n)); CUDA_TRY(ids_sorted.alloc(n)); CUDA_TRY(pos.alloc(n));
  if (n)
    k_degree<<<grid_for(c, n, 256), 256, 0, st>>>(offp, n, deg.p, ids.p, d_bad.p + 1, row_begin, row_end,
                                                  c->ws.hrow.p, c->ws.pieces.p, huge_ctr, max_huge, max_pieces);
  int H = 0;
  // a valid CSR row has fewer than n entries (deduplicated, no self-loop),
  // so the degree sort needs bit_length(n - 1) key bits (22 for RMAT-22:
  // three onesweep passes instead of four). A malformed row with more only
  // changes which endpoint keeps an edge, never that exactly one does.
  int deg_bits = 1;
  while (deg_bits < 32 && ((int64_t)1 << deg_bits) < n) ++deg_bits;
  {
    // one temp buffer for the sort and the per-chunk scans (no reallocation
    // while the pipeline runs: cudaFree would synchronise the device)
    size_t sort_bytes = 0, b1 = 0, b2 = 0;
    long long max_nr = 1;
    for (size_t k = 0; k + 1 < chunk_rows.size(); ++k)
      max_nr = std::max<long long>(max_nr, chunk_rows[k + 1] - chunk_rows[k]);
    if (n)
      cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, deg.p, deg_sorted.p, ids.p,
                                                ids_sorted.p, (int)n, 0, deg_bits, st);
    cub::DeviceScan::ExclusiveScan(nullptr, b1, (long long*)nullptr, (long long*)nullptr, cuda::std::plus<>{},
                                   cub::FutureValue<long long>(nullptr), (int)max_nr, st);
    cub::DeviceScan::ExclusiveScan(nullptr, b2, (int*)nullptr, (int*)nullptr, cuda::std::plus<>{},
                                   cub::FutureValue<int>(nullptr), (int)max_nr, st);
    CUDA_TRY(c->ws.tmp.alloc(std::max(sort_bytes, std::max(b1, b2))));
  }
  if (n) {
    size_t tmp_bytes = c->ws.tmp.n;
    auto& tmp = c->ws.tmp;
    CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(tmp.p, tmp_bytes, deg.p, deg_sorted.p, ids.p,
                                                       ids_sorted.p, (int)n, 0, deg_bits, st));
    // hubs: the first positions with degree >= kHubMinDegree, at most kHubMax
    const int probe = (int)std::min<int64_t>(n, kHubMax);
    std::vector<int> top(probe);
    unsigned long long h_badoff = 0;
    CUDA_TRY(cudaMemcpyAsync(top.data(), deg_sorted.p, sizeof(int) * probe, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&h_badoff, d_bad.p + 1, sizeof h_badoff, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (h_badoff != ~0ull) return fail(FSV_ERR_INPUT, "row_offsets must be non-decreasing");
    int cand = 0;
    while (cand < probe && top[cand] >= kHubMinDegree) ++cand;
    H = (c->hub_limit >= 0) ? std::min(cand, c->hub_limit) : 0;
    H &= ~3;
    if (H < 256) H = 0;
  }
  // L2 rank tier: when the vectors overflow L2 and the degrees are skewed,
  // the next most connected vertices (degree >= kTierMinDegree, at most
  // kTierMax) also get a compact slot, gathered from the L2-resident G_hub
  int HT = H;
  long long tier_min_n = kTierMinN;
  if (const char* env = getenv("FSV_TIER_MIN_N")) tier_min_n = atoll(env);   // tests force the tier
  if (H && n >= tier_min_n && c->hub_limit >= 0) {
    k_count_ge<<<1, 32, 0, st>>>(deg_sorted.p, n, kTierMinDegree, reinterpret_cast<long long*>(d_bad.p + 1));
    long long cnt_ge = 0;
    CUDA_TRY(cudaMemcpyAsync(&cnt_ge, d_bad.p + 1, sizeof cnt_ge, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    const long long t = std::min<long long>(cnt_ge, kTierMax) & ~3LL;
    if (t > H) {
      HT = (int)t;
      if (c->hub_auto) H = std::min(H, kHubAutoTier);
    }
  }
  // column-range tiling (k_tile_pass, fsv_set_tile_width): no hub table, no
  // huge rows, vectors over one tile. Off by default: the tile passes cost
  // more layout time than one solve gains; auto = 8 M vertices
  // (32 MB slices of each vertex vector).
  int T = 1;
  long long tile_w = c->tile_width < 0 ? (8LL << 20) : c->tile_width;
  {
    if (const char* e = getenv("FSV_TILE_W")) tile_w = atoll(e);   // tests/dev: exact width in vertices
    if (tile_w > 0 && n > tile_w) T = (int)((n + tile_w - 1) / tile_w);
  }
  c->tiles = T;
  c->H = H;
  c->HT = HT;
  CUDA_TRY(c->hub_id.alloc((size_t)((std::max(HT, 4) + (1 << 19) - 1) >> 19 << 19)));   // 2 MB multiple
  if (n) k_positions<<<grid_for(c, n, 256), 256, 0, st>>>(ids_sorted.p, n, HT, pos.p, c->hub_id.p);
  umark(1);

  // orientation, chunk by chunk as the columns arrive: encode (one gather
  // per entry), exclusive scans seeded with the running totals of the
  // earlier chunks (device-side carry), compact into the final layout. Only
  // the last chunk's work trails the transfer. ecol is sized by the bound
  // E <= kept entries + headers <= mloc + rows until E is known.
  auto& cnt = c->ws.cnt;
  auto& out_off = c->ws.out_off;
  auto& nzflag = c->ws.nzflag;
  auto& nzidx = c->ws.nzidx;
  auto& etmp = c->ws.etmp;
  auto& nzrows = c->ws.nzrows;
  auto& nzoff = c->ws.nzoff;
  const int K = (int)chunk_rows.size() - 1;
  CUDA_TRY(cnt.alloc(rows + 1)); CUDA_TRY(out_off.alloc(rows + 1));
  CUDA_TRY(nzflag.alloc(rows + 1)); CUDA_TRY(nzidx.alloc(rows + 1));
  CUDA_TRY(etmp.alloc((size_t)std::max<int64_t>(mloc, 1)));
  CUDA_TRY(nzrows.alloc((size_t)rows + 1));
  CUDA_TRY(nzoff.alloc((size_t)rows + 1));
  {
    long long epad = 0;   // dev: FSV_EPAD shifts the layout (placement sensitivity checks)
    if (const char* e = getenv("FSV_EPAD")) epad = atoll(e);
    CUDA_TRY(c->ecol.alloc((size_t)(mloc + rows + SPAN + epad)));
    c->ecolp = c->ecol.p + epad;
  }
  CUDA_TRY(c->ws.carry_e.alloc((size_t)K + 1));
  CUDA_TRY(c->ws.carry_r.alloc((size_t)K + 1));
  CUDA_TRY(cudaMemsetAsync(c->ws.carry_e.p, 0, sizeof(long long), st));
  CUDA_TRY(cudaMemsetAsync(c->ws.carry_r.p, 0, sizeof(int), st));
  umark(2);
  for (int k = 0; k < K; ++k) {
    const long long u0 = chunk_rows[k], u1 = chunk_rows[k + 1], nr = u1 - u0;
    const long long r0 = u0 - row_begin, r1 = u1 - row_begin;
    if (cols_pageable) {
      const int64_t lo = h_off[u0] - e_begin, hi = h_off[u1] - e_begin;
      if (lo < 0 || hi > mloc || hi < lo) return fail(FSV_ERR_INPUT, "row_offsets must be non-decreasing");
      int rc = staged_h2d(c, d_cols.p + lo, h_cols + lo, sizeof(ColT) * (hi - lo), c->copy_stream);
      if (rc) return rc;
      CUDA_TRY(cudaEventRecord(c->chunk_ev[k], c->copy_stream));
    }
    CUDA_TRY(cudaStreamWaitEvent(st, c->chunk_ev[k], 0));
    if (nr) {
      k_orient_encode<ColT><<<grid_for(c, (nr + 31) / 32 * 32, 256, 16), 256, 0, st>>>(
          offp, colp, e_begin, u0, nr, n, pos.p, HT, etmp.p, cnt.p + r0, nzflag.p + r0, d_bad.p);
      k_piece_encode<ColT><<<c->sm_count * 16, 256, 0, st>>>(
          c->ws.pieces.p, huge_ctr + 1, u0, u1, offp, colp, e_begin, n, pos.p, HT, etmp.p,
          c->ws.hkept.p, c->ws.piece_kept.p, d_bad.p);
      k_huge_rows<<<c->sm_count * 2, 256, 0, st>>>(c->ws.hrow.p, huge_ctr, r0, r1, c->ws.hkept.p, cnt.p,
                                                  nzflag.p);
    }
    if (nr) {
      size_t b = c->ws.tmp.n;
      CUDA_TRY(cub::DeviceScan::ExclusiveScan(c->ws.tmp.p, b, cnt.p + r0, out_off.p + r0, cuda::std::plus<>{},
                                              cub::FutureValue<long long>(c->ws.carry_e.p + k), (int)nr, st));
      b = c->ws.tmp.n;
      CUDA_TRY(cub::DeviceScan::ExclusiveScan(c->ws.tmp.p, b, nzflag.p + r0, nzidx.p + r0, cuda::std::plus<>{},
                                              cub::FutureValue<int>(c->ws.carry_r.p + k), (int)nr, st));
    }
    k_chunk_carry<<<1, 1, 0, st>>>(cnt.p, nzflag.p, out_off.p, nzidx.p, r0, r1, c->ws.carry_e.p,
                                   c->ws.carry_r.p, k);
    if (nr) {
      k_orient_compact<<<grid_for(c, (nr + 31) / 32 * 32, 256, 16), 256, 0, st>>>(
          offp, e_begin, u0, nr, etmp.p, out_off.p + r0, nzidx.p + r0, c->ecolp, nzrows.p, nzoff.p);
      k_piece_compact<<<c->sm_count * 16, 256, 0, st>>>(
          c->ws.pieces.p, huge_ctr + 1, u0, u1, offp, e_begin, etmp.p, c->ws.hrow.p, out_off.p,
          c->ws.piece_kept.p, c->ecolp);
    }
    if (udbg) {
      cudaEvent_t e; cudaEventCreate(&e); cudaEventRecord(e, st);
      dbg_enc_ev.push_back(e);
    }
  }
  const int KT = K;   // carry slots used
  umark(3);
  long long E = 0;
  int R = 0;
  unsigned long long h_bad = 0, h_overflow = 0;
  CUDA_TRY(cudaMemcpyAsync(&E, c->ws.carry_e.p + KT, sizeof E, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&R, c->ws.carry_r.p + KT, sizeof R, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&h_bad, d_bad.p, sizeof h_bad, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&h_overflow, huge_ctr + 2, sizeof h_overflow, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (h_overflow) return fail(FSV_ERR_INPUT, "row_offsets must be non-decreasing");
  if (h_bad != ~0ull) {
    // graph.py:71-75 semantics: report an offending entry
    const int64_t e = e_begin + (int64_t)h_bad;
    std::vector<int64_t> hv;
    const int64_t* hp = h_off.h;
    if (!hp) {   // device offsets: fetch them for the message (error path only)
      hv.resize((size_t)n + 1);
      CUDA_TRY(cudaMemcpy(hv.data(), offp, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
      hp = hv.data();
    }
    const int64_t* it = std::upper_bound(hp, hp + n + 1, e);
    const long long u = (long long)(it - hp) - 1;
    long long v = -1;
    if (h_cols) {
      v = (long long)h_cols[h_bad];
    } else {
      ColT cv = 0;
      CUDA_TRY(cudaMemcpy(&cv, colp + h_bad, sizeof(ColT), cudaMemcpyDeviceToHost));
      v = (long long)cv;
    }
    return fail(FSV_ERR_INPUT, "edge (%lld, %lld) out of range for n=%lld", u, v, (long long)n);
  }
  if (T > 1 && R > 0) {
    // tiled layout from the built one (k_tile_runs, stable sort by tile,
    // k_tile_scatter); grow-only workspaces (stream-ordered allocations of
    // this size are returned to the driver at every synchronisation)
    auto& tws = c->ws;
    CUDA_TRY(tws.t_runs.alloc((size_t)R));
    CUDA_TRY(tws.t_base.alloc((size_t)R + 1));
    int* runs = tws.t_runs.p;
    long long* run_base = tws.t_base.p;
    const int rg = grid_for(c, R, 256, 16);
    k_tile_runs<false><<<rg, 256, 0, st>>>(c->ecolp, nzoff.p, nzrows.p, R, E, tile_w, runs, nullptr, nullptr,
                                           nullptr, nullptr, nullptr);
    size_t sb = 0;
    cub::DeviceScan::ExclusiveScan(nullptr, sb, runs, run_base, cuda::std::plus<>{}, 0LL, (int)R, st);
    CUDA_TRY(tws.tmp.alloc(std::max(sb, tws.tmp.n)));
    sb = tws.tmp.n;
    CUDA_TRY(cub::DeviceScan::ExclusiveScan(tws.tmp.p, sb, runs, run_base, cuda::std::plus<>{}, 0LL, (int)R, st));
    long long M = 0;
    int last_runs = 0;
    CUDA_TRY(cudaMemcpyAsync(&M, run_base + R - 1, sizeof M, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&last_runs, runs + R - 1, sizeof last_runs, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    M += last_runs;
    CUDA_TRY(tws.t_key.alloc((size_t)M * 2));
    CUDA_TRY(tws.t_ids.alloc((size_t)M * 2));
    CUDA_TRY(tws.t_len.alloc((size_t)M));
    CUDA_TRY(tws.t_row.alloc((size_t)M));
    CUDA_TRY(tws.t_src.alloc((size_t)M));
    CUDA_TRY(tws.t_seg.alloc((size_t)M * 2));
    uint32_t *key = tws.t_key.p, *key2 = tws.t_key.p + M;
    int *ids = tws.t_ids.p, *ids2 = tws.t_ids.p + M, *len = tws.t_len.p, *row = tws.t_row.p;
    long long *src = tws.t_src.p, *seg = tws.t_seg.p, *out = tws.t_seg.p + M;
    k_tile_runs<true><<<rg, 256, 0, st>>>(c->ecolp, nzoff.p, nzrows.p, R, E, tile_w, nullptr, run_base, key, src,
                                          len, row);
    k_iota<<<grid_for(c, M, 256), 256, 0, st>>>(ids, M);
    int kbits = 1;
    while ((1LL << kbits) < T) ++kbits;
    sb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sb, key, key2, ids, ids2, (int)M, 0, kbits, st);
    size_t sb2 = 0;
    cub::DeviceScan::ExclusiveScan(nullptr, sb2, seg, out, cuda::std::plus<>{}, 0LL, (int)M, st);
    CUDA_TRY(cudaStreamSynchronize(st));   // (the workspace may grow)
    CUDA_TRY(tws.tmp.alloc(std::max(std::max(sb, sb2), tws.tmp.n)));
    sb = tws.tmp.n;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(tws.tmp.p, sb, key, key2, ids, ids2, (int)M, 0, kbits, st));
    k_tile_lens<<<grid_for(c, M, 256), 256, 0, st>>>(ids2, len, M, seg);
    sb = tws.tmp.n;
    CUDA_TRY(cub::DeviceScan::ExclusiveScan(tws.tmp.p, sb, seg, out, cuda::std::plus<>{}, 0LL, (int)M, st));
    const long long E2 = E + (M - R);
    long long epad = 0;
    if (const char* e = getenv("FSV_EPAD")) epad = atoll(e);
    CUDA_TRY(cudaStreamSynchronize(st));   // the run lists are read: the segment arrays may grow now
    CUDA_TRY(tws.etmp2.alloc((size_t)(E2 + SPAN + epad)));   // the tiled layout, swapped in below
    CUDA_TRY(nzrows.alloc((size_t)M + 1));
    CUDA_TRY(nzoff.alloc((size_t)M + 1));
    k_tile_scatter<<<grid_for(c, M, 256, 16), 256, 0, st>>>(c->ecolp, ids2, src, len, row, out, M,
                                                                tws.etmp2.p + epad, nzrows.p, nzoff.p);
    CUDA_TRY(cudaGetLastError());
    std::swap(c->ecol.p, tws.etmp2.p);   // (DBuf owns its pointer: swap the members, never copy)
    std::swap(c->ecol.n, tws.etmp2.n);
    std::swap(c->ecol.cap, tws.etmp2.cap);
    c->ecolp = c->ecol.p + epad;
    E = E2;
    R = (int)M;
  }
  const long long Epad = (E + SPAN - 1) / SPAN * SPAN;
  umark(4);
  k_pad<<<grid_for(c, std::max<long long>(Epad - E, 1), 256), 256, 0, st>>>(c->ecolp, E, Epad, (int)n,
                                                                             nzrows.p, R, nzoff.p);
  // the row open at every task boundary: SPAN entries, or STEP entries for a
  // small layout whose warp tasks are single steps (small_layout())
  const long long nsteps = Epad / STEP;
  const bool small = small_layout(c, Epad);
  const long long ntask = small ? nsteps : Epad / SPAN;
  CUDA_TRY(c->span_row.alloc((size_t)std::max<long long>(ntask, 1)));
  if (ntask)
    k_span_row<<<grid_for(c, ntask, 256), 256, 0, st>>>(nzoff.p, nzrows.p, R + 1, ntask,
                                                         small ? STEP : SPAN, c->span_row.p);
  umark(5);

  // f_1 is computed by every solve (k_f1 in solve_impl), not cached here
  CUDA_TRY(c->f1.alloc((size_t)n + 64));

  // keep the rank's symmetric columns (int32) for sparse iterations
  if constexpr (sizeof(ColT) != 4) {
    CUDA_TRY(c->csr_cols.alloc((size_t)std::max<int64_t>(mloc, 1)));
    if (mloc)
      k_narrow<<<grid_for(c, mloc, 256), 256, 0, st>>>(colp, mloc, c->csr_cols.p);
  }
  c->col_base = e_begin;
  c->csr_local = mloc;
  c->offp = offp;
  if constexpr (sizeof(ColT) == 4)
    c->colsp = reinterpret_cast<const int*>(colp);
  else
    c->colsp = c->csr_cols.p;
  c->var_rows_ready = false;
  c->row_begin = row_begin;
  c->row_end = row_end;

  // solve buffers: n + dummy vertex, padded for 16-byte vector access
  const size_t nv = ((size_t)n + 1 + 63) / 64 * 64;
  // Y (f_k of even k) is f1's buffer: k_first leaves f_1 there without a copy
  long long vpad = 0;   // dev: FSV_VPAD shifts X and G (placement checks)
  if (const char* e = getenv("FSV_VPAD")) vpad = atoll(e) / 4 * 4;
  CUDA_TRY(c->xb.alloc(nv + vpad)); CUDA_TRY(c->gb.alloc(nv + vpad));
  c->X = c->xb.p + vpad; c->Y = c->f1.p; c->G = c->gb.p + vpad;
  // The hot hub arrays get whole 2 MB-aligned allocations (cudaMalloc aligns
  // an allocation of >= 2 MB to 2 MB), like the vertex arrays: the dense
  // hook's time depends on their placement relative to the vertex arrays at
  // sub-2 MB offsets (profiles/r02/placement.txt), and a small
  // allocation would land wherever the allocator's pool puts it.
  constexpr long long kAlign2M = (2LL << 20) / (long long)sizeof(int);
  auto round2m = [&](long long ints) { return (std::max<long long>(ints, 4) + kAlign2M - 1) / kAlign2M * kAlign2M; };
  CUDA_TRY(c->G_hub.alloc((size_t)round2m(HT))); {
    long long hpad = 0;   // dev: FSV_HPAD shifts the hub accumulator (placement checks)
    if (const char* e = getenv("FSV_HPAD")) hpad = atoll(e);
    CUDA_TRY(c->hub_acc.alloc((size_t)round2m(acc_len(HT) + hpad)));
    c->hacc = c->hub_acc.p + hpad;
  }
  CUDA_TRY(c->done.alloc(1)); CUDA_TRY(c->ticket.alloc(1));
  CUDA_TRY(c->partials.alloc((size_t)c->sc_grid * 8));
  {
    const long long want = (std::max<long long>(n / 4, 1) + SC_THREADS - 1) / SC_THREADS;
    c->dgrid = (int)std::max<long long>(1, std::min<long long>(want, c->sc_grid));
    const long long stride_groups = (long long)c->dgrid * SC_THREADS;
    const long long iters = (n / 4 + stride_groups - 1) / stride_groups;
    c->rcap = 4 * 32 * std::max<long long>(iters, 1) + 32;
    const long long warps = (long long)c->dgrid * (SC_THREADS / 32);
    CUDA_TRY(c->dlist.alloc((size_t)(warps * c->rcap)));
    CUDA_TRY(c->dcount.alloc((size_t)warps));
    CUDA_TRY(c->mode.alloc((size_t)kTraceCap + 2));
    CUDA_TRY(c->iterbuf.alloc(4));
    CUDA_TRY(c->tstamp.alloc((size_t)kTraceCap + 2));
    // rows longer than PUSH_BIG: sum of ceil(deg / PUSH_BCHUNK) <= mloc / PUSH_BCHUNK + mloc / PUSH_BIG + 1
    CUDA_TRY(c->chunks.alloc((size_t)(mloc / PUSH_BCHUNK + mloc / PUSH_BIG + 64)));
  }
  CUDA_TRY(c->cnt.alloc((size_t)kTraceCap * NCOUNT));
  umark(6);
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaGetLastError());
  if (udbg) {
    const char* names[] = {"degrees+sort+positions", "(setup)", "chunks (encode..compact)", "readback", "pad+spans",
                           "tail (narrow, allocs)"};
    for (int i = 0; i < 6; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, uev[i], uev[i + 1]);
      fprintf(stderr, "[upload] %-24s %8.3f ms\n", names[i], ms);
    }
    for (size_t k = 0; k < dbg_copy_ev.size(); ++k) {
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, uev[0], dbg_copy_ev[k]);
      if (k < dbg_enc_ev.size()) cudaEventElapsedTime(&b, uev[0], dbg_enc_ev[k]);
      fprintf(stderr, "[upload] chunk %zu copied at %8.3f ms, encoded at %8.3f ms\n", k, a, b);
    }
    for (auto& e : uev) cudaEventDestroy(e);
  }

  if (udbg) {   // layout digest (FNV-1a over ecol, span_row)
    std::vector<uint32_t> h((size_t)Epad);
    cudaMemcpy(h.data(), c->ecolp, sizeof(uint32_t) * Epad, cudaMemcpyDeviceToHost);
    uint64_t d = 1469598103934665603ull;
    for (uint32_t x : h) { d ^= x; d *= 1099511628211ull; }
    fprintf(stderr, "[upload] layout digest %016llx E=%lld R=%d\n", (unsigned long long)d, E, R);
  }
  // int32 copy of the offsets for the per-solve f_1 pass when they fit
  // (half the bytes of its offset stream)
  c->off32 = h_off[n] < (int64_t(1) << 31);
  if (c->off32) {
    CUDA_TRY(c->csr_off32.alloc((size_t)n + 1));
    k_narrow<<<grid_for(c, n + 1, 256), 256, 0, st>>>(offp, n + 1, c->csr_off32.p);
    CUDA_TRY(cudaStreamSynchronize(st));
    CUDA_TRY(cudaGetLastError());
  }
  c->n = n;
  c->m_dir = h_off[n];
  c->E = E;
  c->Epad = Epad;
  c->R = R;
  c->ready = true;
  return FSV_OK;
}

extern "C" int fsv_set_tile_width(fsv_ctx* c, int64_t vertices) {
  if (!c) return fail(FSV_ERR_CONTRACT, "NULL context");
  c->tile_width = vertices;
  return FSV_OK;
}

extern "C" int fsv_set_minority_sweep(fsv_ctx* c, int enable) {
  if (!c) return fail(FSV_ERR_CONTRACT, "NULL context");
  c->minority = enable != 0;
  c->graph_dirty = true;
  return FSV_OK;
}

extern "C" int fsv_set_hub_slots(fsv_ctx* c, int slots) {
  if (!c) return fail(FSV_ERR_CONTRACT, "NULL context");
  c->hub_limit = slots < 0 ? -1 : (slots == 0 ? kHubAuto : std::min(slots, kHubMax));
  c->hub_auto = slots == 0;
  return FSV_OK;
}

extern "C" int fsv_upload_csr(fsv_ctx* c, int64_t n, const int64_t* off, const int32_t* cols,
                              int64_t row_begin, int64_t row_end) {
  return upload_impl<int32_t>(c, n, off, cols, row_begin, row_end);
}

extern "C" int fsv_upload_csr_device(fsv_ctx* c, int64_t n, const int64_t* d_off, const int32_t* d_cols,
                                     int64_t row_begin, int64_t row_end) {
  if (!d_off) return fail(FSV_ERR_CONTRACT, "row_offsets is NULL");
  if (!d_cols) {
    // an empty column slice needs no pointer
    static const int32_t none = 0;
    d_cols = &none;   // never read: the upload checks mloc first
  }
  return upload_impl<int32_t>(c, n, nullptr, nullptr, row_begin, row_end, d_cols, d_off, true, true);
}

extern "C" int fsv_upload_csr64(fsv_ctx* c, int64_t n, const int64_t* off, const int64_t* cols,
                                int64_t row_begin, int64_t row_end) {
  return upload_impl<int64_t>(c, n, off, cols, row_begin, row_end);
}

// Edge list -> CsrGraph on the device (graph.py:55-97), then the layout of
// upload_impl. Pairs go up in chunks on the copy stream while the keys of
// earlier chunks are formed; one radix sort over 2b key bits; unique; CSR.
// Temporaries are stream-ordered allocations returned after the build.
template <typename IdT>
static int upload_edges_impl(fsv_ctx* c, int64_t n, int64_t m, const IdT* h_pairs, int64_t row_begin,
                             int64_t row_end) {
  if (!c) return fail(FSV_ERR_CONTRACT, "NULL context");
  if (n < 0) return fail(FSV_ERR_INPUT, "vertex count must be non-negative, got %lld", (long long)n);
  if (n >= (int64_t)IDMASK) return fail(FSV_ERR_INPUT, "n=%lld exceeds the device id range", (long long)n);
  if (m < 0) return fail(FSV_ERR_CONTRACT, "negative edge count %lld", (long long)m);
  if (m > 0 && !h_pairs) return fail(FSV_ERR_CONTRACT, "pairs is NULL");
  if (row_begin < 0 || row_end < row_begin || row_end > n)
    return fail(FSV_ERR_CONTRACT, "row range [%lld, %lld) invalid for n=%lld", (long long)row_begin,
                (long long)row_end, (long long)n);
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  c->ready = false;
  c->labels_ready = 0;
  c->labeling_ready = false;
  int b = 1;
  while ((1LL << b) < n) ++b;        // ids < n <= 2^b
  const long long m2 = 2 * m;
  IdT* d_pairs = nullptr;
  unsigned long long *ka = nullptr, *kb = nullptr;
  long long* d_cnt = nullptr;        // [0] unique keys, [1] CSR entries
  void* d_tmp = nullptr;
  int* d_full = nullptr;             // all rows' columns when only a row range is kept
  auto release = [&]() {
    if (d_pairs) cudaFreeAsync(d_pairs, st);
    if (ka) cudaFreeAsync(ka, st);
    if (kb) cudaFreeAsync(kb, st);
    if (d_tmp) cudaFreeAsync(d_tmp, st);
    if (d_full) cudaFreeAsync(d_full, st);
    if (d_cnt) cudaFreeAsync(d_cnt, st);
    cudaStreamSynchronize(st);
  };
#define EDGE_TRY(x)                                                              \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      release();                                                                 \
      return fail(FSV_ERR_RUNTIME, "%s: %s", #x, cudaGetErrorString(e_));        \
    }                                                                            \
  } while (0)
  EDGE_TRY(cudaMallocAsync(&d_cnt, 2 * sizeof(long long), st));
  EDGE_TRY(c->ws.bad.alloc(2));
  EDGE_TRY(cudaMemsetAsync(c->ws.bad.p, 0xff, sizeof(unsigned long long), st));
  if (m) {
    EDGE_TRY(cudaMallocAsync(&d_pairs, sizeof(IdT) * m2, st));
    EDGE_TRY(cudaMallocAsync(&ka, sizeof(unsigned long long) * m2, st));
    EDGE_TRY(cudaMallocAsync(&kb, sizeof(unsigned long long) * m2, st));
    // chunked H2D on the copy stream, keys of each chunk as it lands
    const int K = m >= (1LL << 22) ? 8 : 1;
    while (c->chunk_ev.size() < (size_t)K + 1) {
      cudaEvent_t e;
      EDGE_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->chunk_ev.push_back(e);
    }
    EDGE_TRY(cudaEventRecord(c->chunk_ev[K], st));          // allocations ordered before the copies
    EDGE_TRY(cudaStreamWaitEvent(c->copy_stream, c->chunk_ev[K], 0));
    for (int k = 0; k < K; ++k) {
      const long long i0 = m * k / K, i1 = m * (k + 1) / K;
      EDGE_TRY(cudaMemcpyAsync(d_pairs + 2 * i0, h_pairs + 2 * i0, sizeof(IdT) * 2 * (i1 - i0),
                               cudaMemcpyHostToDevice, c->copy_stream));
      EDGE_TRY(cudaEventRecord(c->chunk_ev[k], c->copy_stream));
    }
    for (int k = 0; k < K; ++k) {
      const long long i0 = m * k / K, i1 = m * (k + 1) / K;
      EDGE_TRY(cudaStreamWaitEvent(st, c->chunk_ev[k], 0));
      if (i1 > i0)
        k_edge_keys<IdT><<<grid_for(c, i1 - i0, 256, 16), 256, 0, st>>>(d_pairs, i0, i1, n, b, ka, c->ws.bad.p);
    }
    unsigned long long h_bad = ~0ull;
    EDGE_TRY(cudaMemcpyAsync(&h_bad, c->ws.bad.p, sizeof h_bad, cudaMemcpyDeviceToHost, st));
    EDGE_TRY(cudaStreamSynchronize(st));
    if (h_bad != ~0ull) {
      // graph.py:71-75: the first pair (input order) with an endpoint out of range
      const long long u = (long long)h_pairs[2 * h_bad], v = (long long)h_pairs[2 * h_bad + 1];
      release();
      return fail(FSV_ERR_INPUT, "edge (%lld, %lld) out of range for n=%lld", u, v, (long long)n);
    }
    cudaFreeAsync(d_pairs, st);
    d_pairs = nullptr;
    // sort (2b key bits), unique
    size_t sort_bytes = 0, uniq_bytes = 0;
    cub::DoubleBuffer<unsigned long long> dbuf(ka, kb);
    cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, dbuf, m2, 0, 2 * b, st);
    cub::DeviceSelect::Unique(nullptr, uniq_bytes, ka, kb, d_cnt, m2, st);
    EDGE_TRY(cudaMallocAsync(&d_tmp, std::max(sort_bytes, uniq_bytes), st));
    EDGE_TRY(cub::DeviceRadixSort::SortKeys(d_tmp, sort_bytes, dbuf, m2, 0, 2 * b, st));
    unsigned long long* sorted = dbuf.Current();
    unsigned long long* uniq = dbuf.Alternate();
    EDGE_TRY(cub::DeviceSelect::Unique(d_tmp, uniq_bytes, sorted, uniq, d_cnt, m2, st));
    k_key_count<<<1, 1, 0, st>>>(uniq, d_cnt, b, d_cnt + 1);
    long long M = 0;
    EDGE_TRY(cudaMemcpyAsync(&M, d_cnt + 1, sizeof M, cudaMemcpyDeviceToHost, st));
    EDGE_TRY(cudaStreamSynchronize(st));
    // the CSR: offsets into csr_off, columns into csr_cols (full range) or a
    // temporary from which upload_impl copies this rank's slice
    EDGE_TRY(c->csr_off.alloc((size_t)n + 1));
    int* cols_out = nullptr;
    if (row_begin == 0 && row_end == n) {
      EDGE_TRY(c->csr_cols.alloc((size_t)std::max<long long>(M, 1)));
      cols_out = c->csr_cols.p;
    } else {
      EDGE_TRY(cudaMallocAsync(&d_full, sizeof(int) * std::max<long long>(M, 1), st));
      cols_out = d_full;
    }
    k_csr_from_keys<<<grid_for(c, std::max<long long>(M, n + 1), 256, 16), 256, 0, st>>>(uniq, d_cnt + 1, n, b,
                                                                                     c->csr_off.p, cols_out);
  } else {
    EDGE_TRY(cudaMemsetAsync(d_cnt + 1, 0, sizeof(long long), st));
    EDGE_TRY(c->csr_off.alloc((size_t)n + 1));
    EDGE_TRY(c->csr_cols.alloc(1));
    k_csr_from_keys<<<grid_for(c, n + 1, 256, 16), 256, 0, st>>>(nullptr, d_cnt + 1, n, b, c->csr_off.p,
                                                                 c->csr_cols.p);
  }
  if (ka) { cudaFreeAsync(ka, st); ka = nullptr; }
  if (kb) { cudaFreeAsync(kb, st); kb = nullptr; }
  if (d_tmp) { cudaFreeAsync(d_tmp, st); d_tmp = nullptr; }
  const int32_t* src = d_full ? d_full : c->csr_cols.p;
  const int rc = upload_impl<int32_t>(c, n, nullptr, nullptr, row_begin, row_end, src, c->csr_off.p);
  release();
#undef EDGE_TRY
  return rc;
}

extern "C" int fsv_upload_edges(fsv_ctx* c, int64_t n, int64_t m, const int32_t* pairs, int64_t row_begin,
                                int64_t row_end) {
  return upload_edges_impl<int32_t>(c, n, m, pairs, row_begin, row_end);
}

extern "C" int fsv_upload_edges64(fsv_ctx* c, int64_t n, int64_t m, const int64_t* pairs, int64_t row_begin,
                                  int64_t row_end) {
  return upload_edges_impl<int64_t>(c, n, m, pairs, row_begin, row_end);
}

extern "C" int fsv_get_csr(fsv_ctx* c, int64_t* row_offsets, int32_t* cols, int64_t* csr_entries) {
  if (!c) return fail(FSV_ERR_CONTRACT, "NULL context");
  if (!c->ready) return fail(FSV_ERR_CONTRACT, "no graph uploaded");
  const int64_t mloc = c->csr_local;
  if (csr_entries) *csr_entries = mloc;
  CUDA_TRY(cudaSetDevice(c->device));
  if (row_offsets)
    CUDA_TRY(cudaMemcpyAsync(row_offsets, c->offp, sizeof(int64_t) * (c->n + 1), cudaMemcpyDeviceToHost,
                             c->stream));
  if (cols && mloc)
    CUDA_TRY(cudaMemcpyAsync(cols, c->colsp, sizeof(int32_t) * mloc, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FSV_OK;
}

// ---------------------------------------------------------------------------
// solve

// Buffers of iteration k >= 2: F = f_{k-1}, N = f_k (initialised to gf_{k-1}).
// k_first leaves f_1 in Y and gf_1 in X, so even k reads F = Y, N = X.
static inline int* bufF(fsv_ctx* c, int k) { return (k & 1) ? c->X : c->Y; }
static inline int* bufN(fsv_ctx* c, int k) { return (k & 1) ? c->Y : c->X; }

static constexpr int kPev = 10;  // profile events per iteration

// Vertex-parallel kernels run one resident wave (grid-stride inside): their
// end-of-block counter barrier makes extra waves expensive.
static inline int vertex_grid(fsv_ctx* c) { return c->dgrid; }

static DeltaOut delta_out(fsv_ctx* c) {
  DeltaOut d;
  d.list = c->dlist.p;
  d.count = c->dcount.p;
  d.rcap = c->rcap;
  d.mode = c->mode.p;
  d.policy = c->policy == 1 ? 1 : (c->policy == 2 ? 2 : 0);
  d.threshold = c->threshold;
  d.n_total = c->n;
  return d;
}

static int ensure_pevents(fsv_ctx* c, size_t count) {
  while (c->pev.size() < count) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    c->pev.push_back(e);
  }
  return FSV_OK;
}

static inline void pmark(fsv_ctx* c, int k, int slot) {
  if (c->profile) cudaEventRecord(c->pev[(size_t)k * kPev + slot], c->stream);
}

static LoopCtl loop_ctl(fsv_ctx* c, int graph) {
  LoopCtl l;
  l.iterp = c->iterbuf.p;
  l.cnt_base = c->cnt.p;
  l.tstamp = c->tstamp.p;
  l.cond = (unsigned long long)c->graph_cond;
  l.cond_next = (graph && c->graph_half2) ? (unsigned long long)c->graph_cond_next : 0ull;
  l.rep = graph ? c->rep.p : nullptr;
  l.mode_base = c->mode.p;
  l.graph = graph;
  l.X = c->X;
  l.Y = c->Y;
  return l;
}

// Min-merge of the R partial next-parent vectors of an emulated rank group
// (fsv_group_solve): the elementwise min over ranks is written back to every
// rank's buffer, exactly what ncclAllReduce(ncclInt32, ncclMin) produces in
// the multi-process path. One launch over all ranks' data, no
// kernel waits on another.
constexpr int kGroupMax = 8;
struct MergeArgs {
  int* buf[kGroupMax];
  int count;
  long long n;
  const int* done;   // skip once converged (speculative host-loop launches)
};

__global__ void k_group_min_merge(MergeArgs a) {
  if (a.done && __ldcg(a.done)) return;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n; i += stride) {
    int v = a.buf[0][i];
    for (int r = 1; r < a.count; ++r) v = min(v, a.buf[r][i]);
    for (int r = 0; r < a.count; ++r)
      if (a.buf[r][i] != v) a.buf[r][i] = v;
  }
}

// Queue the hooking phase of iteration k (host loop), or, with graph = true,
// of one half of the graph body whose buffer parity is that of k (the
// iteration number itself is read by the kernels from device memory).
static int launch_hook(fsv_ctx* c, int k, bool graph) {
  cudaStream_t st = c->stream;
  const LoopCtl lc = loop_ctl(c, graph ? 1 : 0);
  if (c->profile) {
    int rc = ensure_pevents(c, (size_t)(k + 1) * kPev);
    if (rc) return rc;
  }
  int* F = bufF(c, k);
  int* N = bufN(c, k);
  // warp tasks: STEPS steps each, or one step when the layout has fewer
  // STEP-entry steps than FSV_SMALL_TASKS x the resident warps (a small graph
  // then spreads over every warp instead of a few long tasks)
  const bool small = small_layout(c, c->Epad);
  const long long nspans = small ? c->Epad / STEP : c->Epad / SPAN;
  {
    HookArgs a;
    a.ecol = c->ecolp; a.nspans = nspans; a.span_row = c->span_row.p;
    a.F = F; a.G = c->G; a.N = N; a.G_hub = c->G_hub.p; a.H = c->H; a.HT = c->HT;
    a.hub_acc = c->hacc; a.hub_id = c->hub_id.p;
    a.done = c->done.p; a.mode = c->mode.p; a.iter = k;
    PushArgs& p = a.push;
    p.list = c->dlist.p; p.count = c->dcount.p; p.rcap = c->rcap;
    p.nregions = c->dgrid * (SC_THREADS / 32);
    p.off = c->offp; p.cols = c->colsp; p.col_base = c->col_base;
    p.row_begin = (int)c->row_begin; p.row_end = (int)c->row_end;
    p.F = F; p.G = c->G; p.N = N; p.mode = c->mode.p; p.iter = k;
    unsigned long long* slot = c->cnt.p + (size_t)(k - 1) * NCOUNT;
    p.flops = slot + C_FLOPS; p.nchunks = slot + C_CHUNKS;
    p.barrier = reinterpret_cast<unsigned*>(slot + C_BARRIER); p.chunks = c->chunks.p;
    a.fix_barrier = reinterpret_cast<unsigned*>(slot + C_FIXBAR);
    a.task_ctr = reinterpret_cast<unsigned*>(slot + C_SPANS);
    a.lc = lc;
    // minority sweep: every rank holds the whole gf vector and all row offsets,
    // so each computes the same global degree sum and takes the same branch;
    // a rank then pushes from the listed vertices of its own rows
    a.n = c->n;
    a.mlist = c->dlist.p; a.mcount = c->dcount.p;
    a.off32 = c->off32 ? c->csr_off32.p : nullptr;
    // (a region must hold one entry per 4-vertex group of its share, which the
    // delta regions' capacity guarantees; vector loads need a 16-byte aligned
    // offset array, which a borrowed one may not be)
    const long long gper = ((c->n + 3) / 4 + p.nregions - 1) / std::max(p.nregions, 1);
    a.minority_thr = (c->minority && c->H && gper <= c->rcap && (uintptr_t)c->offp % 16 == 0)
                         ? c->m_dir / kMinorityDiv : -1;
    // persistent, one CTA per SM; cooperative launch guarantees co-residency
    // for the grid barrier of the sparse (push) path
    pmark(c, k, 0);
    void* kargs[] = {&a};
    const size_t dyn = std::max<size_t>(c->H ? (size_t)(HOT_ACC + c->H) * sizeof(int) : 0,
                                        PUSH_SCRATCH_BYTES);
    const void* fn = small ? (c->HT > c->H ? (const void*)k_hook<true, true, 1>
                              : c->H       ? (const void*)k_hook<true, false, 1>
                                           : (const void*)k_hook<false, false, 1>)
                           : (c->HT > c->H ? (const void*)k_hook<true, true, STEPS>
                              : c->H       ? (const void*)k_hook<true, false, STEPS>
                                           : (const void*)k_hook<false, false, STEPS>);
    CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(c->sm_count), dim3(HOOK_THREADS), kargs, dyn, st));
    pmark(c, k, 1);
    ++c->launches;
  }
  if (c->HT && !FSV_FUSE_HUBFIX) {
    pmark(c, k, 2);
    k_hubfix<<<grid_for(c, c->HT, 256), 256, 0, st>>>(c->hacc, c->hub_id.p, c->G_hub.p, c->HT, N,
                                                       c->done.p, c->mode.p, k,
                                                       graph ? c->iterbuf.p : nullptr, c->X, c->Y);
    pmark(c, k, 3);
    ++c->launches;
  }
  return FSV_OK;
}

// The exchange between the hooking phase and the vertex pass: nothing on one
// rank, ncclAllReduce(min) of the next-parent vector with a communicator, or
// the device min-merge of an emulated rank group.
static int launch_exchange(fsv_ctx* const* cs, int count, int k) {
  fsv_ctx* c = cs[0];
  if (count > 1) {
    MergeArgs m{};
    for (int r = 0; r < count; ++r) m.buf[r] = bufN(cs[r], k);
    m.count = count;
    m.n = c->n;
    m.done = c->done.p;
    if (c->n) {
      k_group_min_merge<<<grid_for(c, c->n, 256), 256, 0, c->stream>>>(m);
      ++c->launches;
    }
    return FSV_OK;
  }
  if (c->comm && c->n) {
    pmark(c, k, 8);
    NCCL_TRY(g_nccl.AllReduce(bufN(c, k), bufN(c, k), (size_t)c->n, ncclInt32, ncclMin, c->comm, c->stream));
    pmark(c, k, 9);
  }
  return FSV_OK;
}

// The vertex pass of iteration k: grandparents, counters, convergence flag.
static int launch_vertex(fsv_ctx* c, int k, int max_iter, bool graph) {
  const LoopCtl lc = loop_ctl(c, graph ? 1 : 0);
  ShortcutArgs s;
  s.F = bufF(c, k); s.G = c->G; s.N = bufN(c, k); s.n = c->n; s.hub_id = c->hub_id.p; s.G_hub = c->G_hub.p;
  s.H = c->HT; s.cnt = c->cnt.p + (size_t)(k - 1) * NCOUNT; s.ticket = c->ticket.p; s.done = c->done.p;
  s.partials = c->partials.p;
  s.dl = delta_out(c);
  s.iter = k; s.max_iter = max_iter;
  s.lc = lc;
  s.mode = c->mode.p;
  pmark(c, k, 6);
  // cooperative: the stochastic hooks of a dense iteration need grid barriers
  void* kargs[] = {&s};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_shortcut, dim3(vertex_grid(c)), dim3(SC_THREADS), kargs, 0,
                                       c->stream));
  pmark(c, k, 7);
  ++c->launches;
  return FSV_OK;
}

static int launch_iteration(fsv_ctx* c, int k, int max_iter, bool graph = false) {
  int rc = launch_hook(c, k, graph);
  if (!rc) rc = launch_exchange(&c, 1, k);
  if (!rc) rc = launch_vertex(c, k, max_iter, graph);
  return rc;
}

// One iteration of an emulated rank group: every rank's hooking phase, the
// device min-merge, every rank's (replicated) vertex pass.
static int launch_group_iteration(fsv_ctx* const* cs, int count, int k, int max_iter) {
  int rc = FSV_OK;
  for (int r = 0; r < count && !rc; ++r) rc = launch_hook(cs[r], k, false);
  if (!rc) rc = launch_exchange(cs, count, k);
  for (int r = 0; r < count && !rc; ++r) rc = launch_vertex(cs[r], k, max_iter, false);
  return rc;
}

// ---- sparse-iteration delta exchange (multi-rank) -----------
// A sparse (push) iteration lowers few entries of N, and N starts as the
// replicated gf_k on every rank (E1), so a rank's contribution to the merged
// N is exactly its entries with N[i] < gf_k[i]. Each rank compacts those
// (i, N[i]) pairs, the lists are all-gathered (ncclAllGather, bytes on the
// wire proportional to the largest list) and every rank min-reduces the other
// ranks' pairs into its N — the same elementwise min the dense allreduce
// computes (the reference's reason for SpMSpV is to move only the delta,
// kernels.py:71-102). Falls back to the allreduce when the
// lists are not smaller.
__global__ void k_delta_compact(const int* __restrict__ N, const int* __restrict__ G, long long n,
                                int2* __restrict__ out, unsigned* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += stride) {   // block-uniform
    const long long i = base + threadIdx.x;
    const bool on = i < n && __ldg(N + i) < __ldg(G + i);
    const unsigned b = __ballot_sync(0xffffffffu, on);
    if (!b) continue;
    unsigned at = 0;
    if (lane == 0) at = atomicAdd(cnt, (unsigned)__popc(b));
    at = __shfl_sync(0xffffffffu, at, 0);
    if (on) out[at + __popc(b & ((1u << lane) - 1u))] = make_int2((int)i, __ldg(N + i));
  }
}

// N <-min the pairs of every other rank: lists[r][0 .. counts[r]) of the
// gathered buffer (cap pairs per rank).
__global__ void k_delta_apply(const int2* __restrict__ all, const unsigned* __restrict__ counts, int nranks,
                              long long cap, int self, int* __restrict__ N) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int r = 0; r < nranks; ++r) {
    if (r == self) continue;
    const long long cr = counts[r];
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < cr; e += stride) {
      const int2 x = all[r * cap + e];
      red_min(N + x.x, x.y);
    }
  }
}

// Emulated group: rank `self`'s N <-min every other rank's list.
struct GroupDelta {
  const int2* list[kGroupMax];
  const unsigned* cnt[kGroupMax];
  int count;
};
__global__ void k_group_delta_apply(GroupDelta a, int self, int* __restrict__ N) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int r = 0; r < a.count; ++r) {
    if (r == self) continue;
    const long long cr = *a.cnt[r];
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < cr; e += stride) {
      const int2 x = a.list[r][e];
      red_min(N + x.x, x.y);
    }
  }
}

static int ensure_delta_buffers(fsv_ctx* c, long long pairs_all) {
  CUDA_TRY(c->dx_list.alloc((size_t)std::max<long long>(c->n, 1)));
  CUDA_TRY(c->dx_cnt.alloc(kGroupMax + 256));
  if (pairs_all > 0) CUDA_TRY(c->dx_all.alloc((size_t)pairs_all));
  if (!c->h_dx_cnt) CUDA_TRY(cudaMallocHost(&c->h_dx_cnt, sizeof(unsigned) * (kGroupMax + 256)));
  return FSV_OK;
}

// Exchange of a sparse iteration k across the group / communicator. Host
// synchronising (the list sizes decide the transfer); all ranks take the same
// branch because they see the same counts.
static int launch_delta_exchange(fsv_ctx* const* cs, int count, int k) {
  fsv_ctx* c = cs[0];
  cudaStream_t st = c->stream;
  const long long n = c->n;
  const int P = count > 1 ? count : c->nranks;
  int rc = FSV_OK;
  for (int r = 0; r < count; ++r) {
    fsv_ctx* x = cs[r];
    if ((rc = ensure_delta_buffers(x, 0))) return rc;
    CUDA_TRY(cudaMemsetAsync(x->dx_cnt.p, 0, sizeof(unsigned) * (kGroupMax + 1), st));
    if (n) k_delta_compact<<<grid_for(x, n, 256), 256, 0, st>>>(bufN(x, k), x->G, n, x->dx_list.p, x->dx_cnt.p);
    ++x->launches;
  }
  unsigned* hc = c->h_dx_cnt;
  if (count > 1) {
    for (int r = 0; r < count; ++r)
      CUDA_TRY(cudaMemcpyAsync(hc + r, cs[r]->dx_cnt.p, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  } else {
    // counts of every rank: one 4-byte allgather
    NCCL_TRY(g_nccl.AllGather(c->dx_cnt.p, c->dx_cnt.p + 1, 1, ncclUint32, c->comm, st));
    CUDA_TRY(cudaMemcpyAsync(hc, c->dx_cnt.p + 1, sizeof(unsigned) * P, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  ++c->host_syncs;
  unsigned cmax = 0;
  for (int r = 0; r < P; ++r) cmax = std::max(cmax, hc[r]);
  // delta only when the gathered lists are smaller than the allreduce's
  // bus bytes per rank (2 (P-1)/P * 4n)
  const double delta_bytes = 8.0 * (double)cmax * (double)P;
  const double dense_bytes = 2.0 * (P - 1) / P * 4.0 * (double)n;
  if (delta_bytes >= dense_bytes) {
    for (int r = 0; r < count; ++r) ++cs[r]->dense_x;
    if (count == 1) c->xbytes += (long long)dense_bytes;
    return launch_exchange(cs, count, k);
  }
  for (int r = 0; r < count; ++r) ++cs[r]->delta_x;
  if (count > 1) {
    GroupDelta gd{};
    gd.count = count;
    for (int r = 0; r < count; ++r) {
      gd.list[r] = cs[r]->dx_list.p;
      gd.cnt[r] = cs[r]->dx_cnt.p;
    }
    for (int r = 0; r < count; ++r) {
      k_group_delta_apply<<<grid_for(c, std::max<long long>(cmax, 1), 256), 256, 0, st>>>(gd, r, bufN(cs[r], k));
      ++c->launches;
    }
    return FSV_OK;
  }
  if (cmax == 0) return FSV_OK;
  if ((rc = ensure_delta_buffers(c, (long long)cmax * P))) return rc;
  NCCL_TRY(g_nccl.AllGather(c->dx_list.p, c->dx_all.p, (size_t)cmax * 2, ncclInt32, c->comm, st));
  k_delta_apply<<<grid_for(c, (long long)cmax * (P - 1), 256), 256, 0, st>>>(c->dx_all.p, c->dx_cnt.p + 1, P,
                                                                             (long long)cmax, c->rank, bufN(c, k));
  ++c->launches;
  c->xbytes += (long long)(8.0 * cmax * (P - 1));
  return FSV_OK;
}

// One iteration of a multi-rank solve with the host in the loop (the
// iteration's product kind is known on the host): dense iterations merge by
// allreduce / device min-merge, sparse ones by the delta exchange.
static int launch_multi_iteration(fsv_ctx* const* cs, int count, int k, int max_iter, bool sparse) {
  int rc = FSV_OK;
  fsv_ctx* c = cs[0];
  for (int r = 0; r < count && !rc; ++r) rc = launch_hook(cs[r], k, false);
  if (rc) return rc;
  pmark(c, k, 8);
  if (sparse) {
    rc = launch_delta_exchange(cs, count, k);
  } else {
    for (int r = 0; r < count; ++r) ++cs[r]->dense_x;
    if (count == 1 && c->comm) c->xbytes += (long long)(2.0 * (c->nranks - 1) / c->nranks * 4.0 * (double)c->n);
    rc = launch_exchange(cs, count, k);
  }
  pmark(c, k, 9);
  for (int r = 0; r < count && !rc; ++r) rc = launch_vertex(cs[r], k, max_iter, false);
  return rc;
}

// The buffers, sizes and launch shapes baked into the captured iteration
// loop. A re-upload that leaves all of them unchanged (the same graph again:
// the workspaces only grow) keeps the instantiated graph.
static std::vector<long long> graph_key(const fsv_ctx* c) {
  auto P = [](const void* p) { return (long long)(uintptr_t)p; };
  return {P(c->ecolp), c->Epad, P(c->span_row.p), P(c->X), P(c->Y), P(c->G), P(c->G_hub.p), c->H, c->HT,
          P(c->hacc), P(c->hub_id.p), P(c->done.p), P(c->mode.p), P(c->dlist.p), P(c->dcount.p), c->rcap,
          c->dgrid, P(c->offp), P(c->colsp), c->col_base, c->row_begin, c->row_end, P(c->cnt.p),
          P(c->chunks.p), P(c->iterbuf.p), P(c->tstamp.p), P(c->ticket.p), P(c->partials.p), c->n,
          c->sm_count, P(c->comm), c->minority, P(c->off32 ? c->csr_off32.p : nullptr)};
}

// Builds (or reuses) the CUDA graph of the iteration loop: one conditional
// WHILE node whose body is an even and an odd iteration (buffer parity).
static int ensure_graph(fsv_ctx* c, int cap) {
  if (c->graph_dirty && c->graph_exec && graph_key(c) == c->graph_key) c->graph_dirty = false;
  if (!c->graph_dirty && c->graph_exec && c->graph_key_policy == c->policy &&
      c->graph_key_thr == c->threshold && c->graph_key_cap == cap)
    return FSV_OK;
  if (c->graph_exec) { cudaGraphExecDestroy(c->graph_exec); c->graph_exec = nullptr; }
  if (c->graph) { cudaGraphDestroy(c->graph); c->graph = nullptr; }
  CUDA_TRY(cudaGraphCreate(&c->graph, 0));
  CUDA_TRY(cudaGraphConditionalHandleCreate(&c->graph_cond, c->graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = c->graph_cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CUDA_TRY(cudaGraphAddNode(&node, c->graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  const bool prof = c->profile;
  c->profile = false;
  int rc = FSV_OK;
#if FSV_GRAPH_IF
  // body = iteration A, then IF(A did not stop) { iteration B }: two
  // iterations per body pass without launching B's kernels after the last
  // iteration (A's vertex pass sets the IF condition with the loop's)
  CUDA_TRY(cudaGraphConditionalHandleCreate(&c->graph_cond_next, body, 0, cudaGraphCondAssignDefault));
  c->graph_half2 = true;
  CUDA_TRY(cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  rc = launch_iteration(c, 2, cap, true);
  {
    cudaGraph_t captured = body;
    const cudaError_t ec = cudaStreamEndCapture(c->stream, &captured);
    c->graph_half2 = false;
    if (rc) { c->profile = prof; return rc; }
    CUDA_TRY(ec);
  }
  // the IF node depends on every leaf of the captured first iteration
  size_t nn = 0;
  CUDA_TRY(cudaGraphGetNodes(body, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn), leaves;
  CUDA_TRY(cudaGraphGetNodes(body, nodes.data(), &nn));
  for (cudaGraphNode_t nd : nodes) {
    size_t nd_out = 0;
    CUDA_TRY(cudaGraphNodeGetDependentNodes(nd, nullptr, &nd_out));
    if (nd_out == 0) leaves.push_back(nd);
  }
  cudaGraphNodeParams ip = {};
  ip.type = cudaGraphNodeTypeConditional;
  ip.conditional.handle = c->graph_cond_next;
  ip.conditional.type = cudaGraphCondTypeIf;
  ip.conditional.size = 1;
  cudaGraphNode_t ifnode;
  CUDA_TRY(cudaGraphAddNode(&ifnode, body, leaves.data(), leaves.size(), &ip));
  cudaGraph_t body2 = ip.conditional.phGraph_out[0];
  CUDA_TRY(cudaStreamBeginCaptureToGraph(c->stream, body2, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  rc = launch_iteration(c, 3, cap, true);
  {
    cudaGraph_t captured = body2;
    const cudaError_t ec = cudaStreamEndCapture(c->stream, &captured);
    c->profile = prof;
    if (rc) return rc;
    CUDA_TRY(ec);
  }
#else
  CUDA_TRY(cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0,
                                         cudaStreamCaptureModeRelaxed));
  // FSV_GRAPH_BODY iterations per body pass (kernels pick their buffers by
  // the device-side iteration number; iterations past convergence exit at
  // once, which is cheaper than relaunching the body)
  for (int k = 2; k < 2 + FSV_GRAPH_BODY && !rc; ++k) rc = launch_iteration(c, k, cap, true);
  cudaGraph_t captured = body;
  const cudaError_t ec = cudaStreamEndCapture(c->stream, &captured);
  c->profile = prof;
  if (rc) return rc;
  CUDA_TRY(ec);
#endif
  CUDA_TRY(cudaGraphInstantiate(&c->graph_exec, c->graph, 0));
  c->graph_dirty = false;
  c->graph_key = graph_key(c);
  c->graph_key_policy = c->policy;
  c->graph_key_thr = c->threshold;
  c->graph_key_cap = cap;
  return FSV_OK;
}

// Copies f_k (the committed parent vector of iteration k) to host.
static int copy_snapshot(fsv_ctx* c, int k, int32_t* dst) {
  const int* src = (k == 1) ? c->Y : bufN(c, k);
  CUDA_TRY(cudaMemcpyAsync(dst, src, sizeof(int) * c->n, cudaMemcpyDeviceToHost, c->stream));
  return FSV_OK;
}

// HookingConfig variants and simplified_sv (fsv_variants.cuh): a host-driven
// loop of init -> hook -> [shortcut] -> commit count per iteration, with the
// reference's stop rule (gf stability only with all four flags,
// algorithms.py:103-114; f stability otherwise, :139).
template <bool STO, bool AGG, bool GP>
static void launch_var_hook(fsv_ctx* c, const int* F, const int* G, int* N) {
  const long long m = c->csr_local;
  if (m)
    k_var_hook<STO, AGG, GP><<<grid_for(c, m, 256, 16), 256, 0, c->stream>>>(c->var_rows.p, c->colsp, m, F,
                                                                              G, N);
}

static int solve_variant(fsv_ctx* c, const fsv_config& d, int cap, int32_t* snapshots, int32_t snap_cap) {
  if (c->comm || c->row_begin != 0 || c->row_end != c->n)
    return fail(FSV_ERR_CONTRACT, "hooking variants run on a single context owning all rows");
  const int fl = d.hooking & 15;
  const bool GP = fl & FSV_HOOK_GRANDPARENT, STO = fl & FSV_HOOK_STOCHASTIC, AGG = fl & FSV_HOOK_AGGRESSIVE;
  const bool gf_stop = (fl & 15) == 15;   // _uses_gf_termination (algorithms.py:103-114)
  cudaStream_t st = c->stream;
  const long long n = c->n;
  c->variant = true;
  c->launches = 0;
  c->host_syncs = 0;
  if (!c->var_rows_ready) {
    CUDA_TRY(c->var_rows.alloc((size_t)std::max<long long>(c->csr_local, 1)));
    if (c->csr_local)
      k_row_ids<<<grid_for(c, n * 32, 256, 16), 256, 0, st>>>(c->offp, c->col_base, 0, n, c->var_rows.p);
    c->var_rows_ready = true;
  }
  const size_t nv = (size_t)n + 64;
  CUDA_TRY(c->var_t.alloc(nv));
  CUDA_TRY(c->var_g.alloc(nv));
  int* P[5] = {c->X, c->G, c->Y, c->var_t.p, c->var_g.p};   // F, G, N, T, Gn
  CUDA_TRY(cudaMemsetAsync(c->cnt.p, 0, sizeof(unsigned long long) * NCOUNT * (size_t)cap, st));
  {
    int rc = ensure_events(c, 3);   // start + two alternating iteration ends
    if (rc) return rc;
  }
  const int vgrid = grid_for(c, n, 256, 8);
  CUDA_TRY(cudaEventRecord(c->events[0], st));
  if (n) k_var_iota<<<vgrid, 256, 0, st>>>(P[0], P[1], n);
  int k = 0;
  bool stopped = false;
  std::vector<float> ms;
  unsigned long long h[NCOUNT];
  cudaEvent_t prev = c->events[0];
  while (k < cap) {
    ++k;
    int* F = P[0];
    int* G = P[1];
    int* N = P[2];
    unsigned long long* cnt = c->cnt.p + (size_t)(k - 1) * NCOUNT;
    if (n) {
      k_var_init<<<vgrid, 256, 0, st>>>(F, G, N, n, STO);
      switch ((STO ? 4 : 0) | (AGG ? 2 : 0) | (GP ? 1 : 0)) {
        case 0: launch_var_hook<false, false, false>(c, F, G, N); break;
        case 1: launch_var_hook<false, false, true>(c, F, G, N); break;
        case 2: launch_var_hook<false, true, false>(c, F, G, N); break;
        case 3: launch_var_hook<false, true, true>(c, F, G, N); break;
        case 4: launch_var_hook<true, false, false>(c, F, G, N); break;
        case 5: launch_var_hook<true, false, true>(c, F, G, N); break;
        case 6: launch_var_hook<true, true, false>(c, F, G, N); break;
        default: launch_var_hook<true, true, true>(c, F, G, N); break;
      }
      if (!STO) k_var_shortcut<<<vgrid, 256, 0, st>>>(N, P[3], n);
      k_var_count<<<vgrid, 256, 0, st>>>(STO ? N : P[3], F, G, P[4], n, cnt);
      c->launches += STO ? 3 : 4;
    }
    cudaEvent_t ev = c->events[1 + (k & 1)];
    CUDA_TRY(cudaEventRecord(ev, st));
    CUDA_TRY(cudaMemcpyAsync(h, cnt, sizeof h, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    ++c->host_syncs;
    float t = 0.f;
    cudaEventElapsedTime(&t, prev, ev);
    ms.push_back(t);
    prev = ev;
    // commit: the new parents become F, their grandparents G
    int* Pn = STO ? P[2] : P[3];
    int* newP[5] = {Pn, P[4], STO ? P[3] : P[2], P[0], P[1]};
    for (int i = 0; i < 5; ++i) P[i] = newP[i];
    if (snapshots) {
      if (k > snap_cap) return fail(FSV_ERR_CONTRACT, "more than %d iterations ran", snap_cap);
      if (n) CUDA_TRY(cudaMemcpyAsync(snapshots + (size_t)(k - 1) * n, P[0], sizeof(int) * n,
                                      cudaMemcpyDeviceToHost, st));
    }
    if (h[C_VIOL]) return fail(FSV_ERR_INVARIANT, "parent vector increased during hooking");
    if ((gf_stop ? h[C_GF] : h[C_F]) == 0) { stopped = true; break; }
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  if (!stopped) return fail(FSV_ERR_RUNTIME, "did not converge within %d iterations", cap);
  c->iterations = k;
  c->h_cnt.assign((size_t)k * NCOUNT, 0ull);
  CUDA_TRY(cudaMemcpy(c->h_cnt.data(), c->cnt.p, sizeof(unsigned long long) * k * NCOUNT, cudaMemcpyDeviceToHost));
  c->h_mode.assign((size_t)k + 1, 0);
  c->iter_ms = ms;
  c->solve_ms = 0.f;
  for (float x : ms) c->solve_ms += x;
  c->components = (int)c->h_cnt[(size_t)(k - 1) * NCOUNT + C_ROOTS];
  c->labels_src = P[0];
  c->labels_ready = 1;
  if (c->h_cnt[(size_t)(k - 1) * NCOUNT + C_NONSTAR])
    return fail(FSV_ERR_INVARIANT, "algorithm terminated on non-star forest");
  return FSV_OK;
}

static int solve_body(fsv_ctx* const* cs, int count, const fsv_config* cfg, int32_t* snapshots,
                      int32_t snap_cap);

// Checked builds clear the registered ranges after every solve, so upload
// kernels (which read other buffers through the same helpers) are unchecked.
static int solve_impl_group(fsv_ctx* const* cs, int count, const fsv_config* cfg, int32_t* snapshots,
                            int32_t snap_cap) {
  const int rc = solve_body(cs, count, cfg, snapshots, snap_cap);
#ifdef FSV_CHECKS
  if (cs && cs[0]) {
    const ChkRanges none{};
    cudaMemcpyToSymbol(g_chk, &none, sizeof none);
  }
#endif
  return rc;
}

static int solve_impl(fsv_ctx* c, const fsv_config* cfg, int32_t* snapshots, int32_t snap_cap) {
  return solve_impl_group(&c, 1, cfg, snapshots, snap_cap);
}

// A rank group runs every rank's kernels on rank 0's stream, in order; the
// contexts' own streams are restored afterwards.
struct StreamGuard {
  fsv_ctx* const* cs;
  int count;
  cudaStream_t saved[kGroupMax];
  StreamGuard(fsv_ctx* const* cs_, int count_) : cs(cs_), count(count_) {
    for (int r = 0; r < count; ++r) {
      saved[r] = cs[r]->stream;
      cs[r]->stream = cs[0]->stream;
    }
  }
  ~StreamGuard() {
    for (int r = 0; r < count; ++r) cs[r]->stream = saved[r];
  }
};

// The group must be one graph split into disjoint row ranges covering
// [0, n) on one device (the 1D partition of SURVEY §8e).
static int check_group(fsv_ctx* const* cs, int count) {
  if (count < 1 || count > kGroupMax) return fail(FSV_ERR_CONTRACT, "group size %d not in 1..%d", count, kGroupMax);
  for (int r = 0; r < count; ++r) {
    if (!cs[r]) return fail(FSV_ERR_CONTRACT, "NULL context");
    if (!cs[r]->ready) return fail(FSV_ERR_CONTRACT, "no graph uploaded");
  }
  if (count == 1) return FSV_OK;
  std::vector<std::pair<int64_t, int64_t>> ranges;
  for (int r = 0; r < count; ++r) {
    const fsv_ctx* c = cs[r];
    for (int q = 0; q < r; ++q)
      if (cs[q] == c) return fail(FSV_ERR_CONTRACT, "a context appears twice in the group");
    if (c->device != cs[0]->device) return fail(FSV_ERR_CONTRACT, "group contexts must share one device");
    if (c->n != cs[0]->n) return fail(FSV_ERR_CONTRACT, "group contexts must hold the same graph (n differs)");
    if (c->comm) return fail(FSV_ERR_CONTRACT, "group contexts cannot carry a communicator");
    ranges.emplace_back(c->row_begin, c->row_end);
  }
  std::sort(ranges.begin(), ranges.end());
  int64_t at = 0;
  for (auto& rg : ranges) {
    if (rg.first != at) return fail(FSV_ERR_CONTRACT, "group row ranges must be disjoint and cover [0, n)");
    at = rg.second;
  }
  if (at != cs[0]->n) return fail(FSV_ERR_CONTRACT, "group row ranges must be disjoint and cover [0, n)");
  return FSV_OK;
}

static int solve_body(fsv_ctx* const* cs, int count, const fsv_config* cfg, int32_t* snapshots,
                      int32_t snap_cap) {
  if (!cs || !cs[0]) return fail(FSV_ERR_CONTRACT, "NULL context");
  int rc = check_group(cs, count);
  if (rc) return rc;
  fsv_ctx* c = cs[0];
  CUDA_TRY(cudaSetDevice(c->device));
  fsv_config d{};
  if (cfg) d = *cfg;
  if (d.max_iters < 0 || d.batch < 0) return fail(FSV_ERR_CONTRACT, "negative max_iters/batch");
  const int cap = d.max_iters > 0 ? std::min(d.max_iters, kTraceCap) : kTraceCap;
  int batch = d.batch > 0 ? d.batch : 4;
  if (snapshots) batch = 1;
  if (d.sparse_policy < 0 || d.sparse_policy > 3)
    return fail(FSV_ERR_CONTRACT, "sparse_policy must be 0..3");
  if (d.sparse_policy == 3 && !(d.sparse_threshold >= 0.0 && d.sparse_threshold <= 1.0))
    return fail(FSV_ERR_CONTRACT, "sparse_threshold must be in [0, 1]");
  if (count > 1 && d.hooking) return fail(FSV_ERR_CONTRACT, "hooking variants run on a single context");
  if (count > 1 && d.profile) return fail(FSV_ERR_CONTRACT, "profile is not supported for rank groups");
  if ((rc = ensure_events(c, 2))) return rc;
  for (int r = 0; r < count; ++r) {
    fsv_ctx* x = cs[r];
    x->launches = 0;
    x->host_syncs = 0;
    x->labels_ready = 0;
    x->labeling_ready = false;
    x->profile = d.profile != 0;
    x->policy = d.sparse_policy;
    x->threshold = d.sparse_policy == 3 ? d.sparse_threshold : 0.1;
    x->hook_ms = x->hubfix_ms = x->shortcut_ms = x->first_ms = x->allreduce_ms = x->push_ms = 0.f;
    x->hook_launches = 0;
  }
  if (d.hooking) {
    if ((d.hooking & ~(FSV_HOOKING_SET | 15)) || !(d.hooking & FSV_HOOKING_SET))
      return fail(FSV_ERR_CONTRACT, "hooking must be 0 or FSV_HOOKING_SET | flag bits, got 0x%x", d.hooking);
    return solve_variant(c, d, cap, snapshots, snap_cap);
  }
  StreamGuard guard(cs, count);
  cudaStream_t st = c->stream;
  for (int r = 0; r < count; ++r) {
    cs[r]->variant = false;
    cs[r]->labels_src = cs[r]->G;
  }
#ifdef FSV_CHECKS
  {  // checked build: the buffers the solve kernels may load from / reduce into (every rank's)
    ChkRanges r{};
    auto add_ld = [&](const int* p, size_t len) { if (p && r.nl < kChkLd) { r.lo[r.nl] = p; r.hi[r.nl++] = p + len; } };
    auto add_red = [&](const int* p, size_t len) {
      if (p && r.nr < kChkRed) { r.rlo[r.nr] = p; r.rhi[r.nr++] = p + len; }
    };
    for (int q = 0; q < count; ++q) {
      const fsv_ctx* x = cs[q];
      add_red(x->xb.p, x->xb.n); add_red(x->f1.p, x->f1.n); add_red(x->hacc, (size_t)acc_len(x->HT));
      add_ld(x->xb.p, x->xb.n); add_ld(x->f1.p, x->f1.n); add_ld(x->gb.p, x->gb.n);
      add_ld(x->G_hub.p, x->G_hub.n); add_ld(x->hub_id.p, x->hub_id.n); add_ld(x->colsp, (size_t)x->csr_local);
      add_ld(x->span_row.p, x->span_row.n);
    }
    CUDA_TRY(cudaMemcpyToSymbolAsync(g_chk, &r, sizeof r, 0, cudaMemcpyHostToDevice, st));
  }
#endif
  if (c->profile && (rc = ensure_pevents(c, 2 * kPev))) return rc;

  // graph mode: the whole iteration loop is one conditional-WHILE graph launch
  // (a communicator's ncclAllReduce is captured into the loop body too: every
  // rank runs the same iterations since the convergence flag is replicated;
  // if NCCL refuses capture into the conditional body, the host loop runs)
  if (d.exchange < 0 || d.exchange > 1) return fail(FSV_ERR_CONTRACT, "exchange must be 0 or 1");
  const bool delta = d.exchange == 0;
  bool graph_mode = count == 1 && c->use_graph && !snapshots && !c->profile && d.batch == 0 &&
                    (!c->comm || c->nranks == 1 || (!c->graph_comm_failed && !delta));
  if (graph_mode && (rc = ensure_graph(c, cap))) {
    if (!c->comm) return rc;
    cudaGetLastError();
    c->graph_comm_failed = true;
    graph_mode = false;
    rc = FSV_OK;
  }
  CUDA_TRY(cudaEventRecord(c->events[0], st));
  for (int r = 0; r < count; ++r) {
    fsv_ctx* x = cs[r];
    k_solve_init<<<grid_for(x, std::max<long long>(x->HT, (long long)cap * NCOUNT), 256), 256, 0, st>>>(
        x->X, x->Y, x->G, x->n, x->hacc, x->HT, x->cnt.p, (long long)cap * NCOUNT, x->done.p,
        x->ticket.p, x->mode.p, x->policy == 2 ? 1 : 0, x->tstamp.p, x->rep.p);
  }
  pmark(c, 1, 6);
  // iteration 1 in closed form: f_1[u] = min(u, smallest neighbour) from the
  // resident CSR rows (first column of each sorted row), every solve; a
  // partitioned graph assembles it from the ranks' rows by a min-merge
  const bool dist = c->comm != nullptr || count > 1;
  if (c->n && !dist && c->row_begin == 0 && c->row_end == c->n) {
    if (c->off32)
      k_f1_solve<int><<<grid_for(c, c->n / 4 + 1, 256, 32), 256, 0, st>>>(c->csr_off32.p, c->colsp,
                                                                        c->n, c->f1.p);
    else
      k_f1_solve<int64_t><<<grid_for(c, c->n / 4 + 1, 256, 32), 256, 0, st>>>(c->offp, c->colsp,
                                                                            c->n, c->f1.p);
    ++c->launches;
  } else if (c->n) {
    for (int r = 0; r < count; ++r) {
      fsv_ctx* x = cs[r];
      k_f1<int><<<grid_for(x, x->n, 256, 64), 256, 0, st>>>(x->offp, x->colsp, x->col_base,
                                                        x->row_begin, x->row_end, x->n, x->f1.p, dist);
      ++x->launches;
    }
    if (c->comm) {
      NCCL_TRY(g_nccl.AllReduce(c->f1.p, c->f1.p, (size_t)c->n, ncclInt32, ncclMin, c->comm, st));
    } else if (count > 1) {
      MergeArgs m{};
      for (int r = 0; r < count; ++r) m.buf[r] = cs[r]->f1.p;
      m.count = count;
      m.n = c->n;
      m.done = nullptr;
      k_group_min_merge<<<grid_for(c, c->n, 256), 256, 0, st>>>(m);
      ++c->launches;
    }
    if (dist)
      for (int r = 0; r < count; ++r) {
        k_f1_fix<<<grid_for(cs[r], cs[r]->n, 256), 256, 0, st>>>(cs[r]->f1.p, cs[r]->n);
        ++cs[r]->launches;
      }
  }
  for (int r = 0; r < count; ++r) {
    fsv_ctx* x = cs[r];
    FirstArgs fa;
    fa.f1 = x->f1.p; fa.G = x->G; fa.X = x->X; fa.n = x->n;
    fa.hub_id = x->hub_id.p; fa.G_hub = x->G_hub.p; fa.H = x->HT; fa.cnt = x->cnt.p;
    fa.partials = x->partials.p; fa.ticket = x->ticket.p; fa.done = x->done.p; fa.max_iter = cap;
    fa.dl = delta_out(x);
    fa.lc = loop_ctl(x, graph_mode ? 2 : 0);
    k_first<<<vertex_grid(x), SC_THREADS, 0, st>>>(fa);
    x->launches += 2;
  }
  pmark(c, 1, 7);
  if ((rc = ensure_events(c, 2))) return rc;
  CUDA_TRY(cudaEventRecord(c->events[1], st));
  if (snapshots) {
    if (snap_cap < 1) return fail(FSV_ERR_CONTRACT, "snapshot capacity exhausted");
    if ((rc = copy_snapshot(c, 1, snapshots))) return rc;
  }
  int launched = 1;  // iterations queued so far (k_first is iteration 1)
  int done = 0;
  int staged = 0;    // iterations whose counters/kinds/stamps are already on the host
  if (graph_mode) {
    CUDA_TRY(cudaGraphLaunch(c->graph_exec, st));
    // end of the device work (events[2] is free in graph mode: iterations
    // >= 2 are timed by %globaltimer stamps)
    if ((rc = ensure_events(c, 3))) return rc;
    CUDA_TRY(cudaEventRecord(c->events[2], st));
    CUDA_TRY(cudaMemcpyAsync(c->h_rep, c->rep.p, sizeof(SolveReport), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    ++c->host_syncs;
    done = c->h_rep->done;
    staged = c->h_rep->iters;   // 0: more than STAGE_ITERS iterations, copied below
    if (done == 0) return fail(FSV_ERR_RUNTIME, "graph loop ended without convergence");
    {
      // kernels the graph ran: iterations 2..it, rounded up to whole body
      // passes unless the IF node skips a pass's second iteration
      const int it = done > 0 ? done : -done;
      const int per_it = 2 + (c->HT && !FSV_FUSE_HUBFIX ? 1 : 0);
      const int passes = std::max(1, (it - 1 + FSV_GRAPH_BODY - 1) / FSV_GRAPH_BODY);
      c->launches += (FSV_GRAPH_IF ? std::max(1, it - 1) : passes * FSV_GRAPH_BODY) * per_it;
    }
  }
  // multi-rank solves keep the host in the loop one iteration at a time:
  // the next iteration's product kind (written by the vertex pass) decides
  // its exchange (dense allreduce or sparse delta lists)
  const bool multi = !graph_mode && (count > 1 || (c->comm && c->nranks > 1));
  for (int r = 0; r < count; ++r) {
    cs[r]->xbytes = 0;
    cs[r]->delta_x = cs[r]->dense_x = 0;
  }
  while (!graph_mode && multi) {
    int hm[2] = {0, 0};
    CUDA_TRY(cudaMemcpyAsync(c->h_done, c->done.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&hm[0], c->mode.p + launched + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    ++c->host_syncs;
    done = *c->h_done;
    if (snapshots && launched > 1) {
      if (launched > snap_cap) return fail(FSV_ERR_CONTRACT, "more than %d iterations ran", snap_cap);
      if ((rc = copy_snapshot(c, launched, snapshots + (size_t)(launched - 1) * c->n))) return rc;
    }
    if (done != 0) break;
    if (launched >= cap) return fail(FSV_ERR_RUNTIME, "did not converge within %d iterations", cap);
    const int k = ++launched;
    if ((rc = launch_multi_iteration(cs, count, k, cap, delta && hm[0] == 1))) return rc;
    if ((rc = ensure_events(c, (size_t)k + 1))) return rc;
    CUDA_TRY(cudaEventRecord(c->events[k], st));
  }
  bool first_round = true;
  while (!graph_mode && !multi) {
    // the first round also holds iteration 1, so it queues batch-1 more
    const int more = first_round ? batch - 1 : batch;
    first_round = false;
    const int upto = std::min(cap, launched + more);
    for (int k = launched + 1; k <= upto; ++k) {
      if ((rc = launch_group_iteration(cs, count, k, cap))) return rc;
      if ((rc = ensure_events(c, (size_t)k + 1))) return rc;
      CUDA_TRY(cudaEventRecord(c->events[k], st));
    }
    launched = std::max(launched, upto);
    CUDA_TRY(cudaMemcpyAsync(c->h_done, c->done.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    ++c->host_syncs;
    done = *c->h_done;
    if (snapshots && (done == 0 || done == launched)) {
      // batch == 1: iteration `launched` has committed f_k
      if (launched > 1) {
        if (launched > snap_cap) return fail(FSV_ERR_CONTRACT, "more than %d iterations ran", snap_cap);
        if ((rc = copy_snapshot(c, launched, snapshots + (size_t)(launched - 1) * c->n))) return rc;
      }
    }
    if (done != 0) break;
    if (launched >= cap)
      return fail(FSV_ERR_RUNTIME, "did not converge within %d iterations", cap);
  }
  if (!graph_mode) CUDA_TRY(cudaStreamSynchronize(st));   // (graph mode synchronised above)
  CUDA_TRY(cudaGetLastError());
  if (done < 0) return fail(FSV_ERR_RUNTIME, "did not converge within %d iterations", -done);
  const int iters = done;
  CUDA_TRY(cudaEventElapsedTime(&c->solve_ms, c->events[0], c->events[graph_mode ? 2 : iters]));
  for (int r = 0; r < count; ++r) {
    fsv_ctx* x = cs[r];
    int xdone = done;
    if (r > 0) {
      CUDA_TRY(cudaMemcpy(&xdone, x->done.p, sizeof(int), cudaMemcpyDeviceToHost));
      if (xdone != done)
        return fail(FSV_ERR_INVARIANT, "rank %d stopped at iteration %d, rank 0 at %d", r, xdone, done);
    }
    x->iterations = iters;
    x->solve_ms = c->solve_ms;
    x->h_cnt.assign((size_t)iters * NCOUNT, 0ull);
    x->h_mode.assign((size_t)iters + 1, 0);
    std::vector<unsigned long long> ts((size_t)iters + 1, 0ull);
    if (graph_mode && iters <= staged) {
      std::copy(x->h_rep->cnt, x->h_rep->cnt + (size_t)iters * NCOUNT, x->h_cnt.begin());
      std::copy(x->h_rep->mode, x->h_rep->mode + iters + 1, x->h_mode.begin());
      std::copy(x->h_rep->ts, x->h_rep->ts + iters + 1, ts.begin());
    } else {
      CUDA_TRY(cudaMemcpy(x->h_cnt.data(), x->cnt.p, sizeof(unsigned long long) * iters * NCOUNT,
                          cudaMemcpyDeviceToHost));
      CUDA_TRY(cudaMemcpy(x->h_mode.data(), x->mode.p, sizeof(int) * (iters + 1), cudaMemcpyDeviceToHost));
      CUDA_TRY(cudaMemcpy(ts.data(), x->tstamp.p, sizeof(unsigned long long) * (iters + 1),
                          cudaMemcpyDeviceToHost));
    }
    x->iter_ms.assign(iters, 0.f);
    for (int k = 1; k <= iters; ++k) x->iter_ms[k - 1] = (float)((double)(ts[k] - ts[k - 1]) * 1e-6);
    x->components = (int)x->h_cnt[(size_t)(iters - 1) * NCOUNT + C_ROOTS];
    x->labels_ready = 1;
  }
  // the pushed-entry count (trace flops of a sparse iteration) is rank-local:
  // every rank reports the group's sum
  if (count > 1)
    for (int k = 0; k < iters; ++k) {
      unsigned long long sum = 0;
      for (int r = 0; r < count; ++r) sum += cs[r]->h_cnt[(size_t)k * NCOUNT + C_FLOPS];
      for (int r = 0; r < count; ++r) cs[r]->h_cnt[(size_t)k * NCOUNT + C_FLOPS] = sum;
    }
  if (c->comm && c->nranks > 1 && iters > 0) {
    DBuf<unsigned long long> fl;
    CUDA_TRY(fl.alloc((size_t)iters));
    std::vector<unsigned long long> h((size_t)iters);
    for (int k = 0; k < iters; ++k) h[(size_t)k] = c->h_cnt[(size_t)k * NCOUNT + C_FLOPS];
    CUDA_TRY(cudaMemcpyAsync(fl.p, h.data(), sizeof(unsigned long long) * iters, cudaMemcpyHostToDevice, st));
    NCCL_TRY(g_nccl.AllReduce(fl.p, fl.p, (size_t)iters, ncclUint64, ncclSum, c->comm, st));
    CUDA_TRY(cudaMemcpyAsync(h.data(), fl.p, sizeof(unsigned long long) * iters, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int k = 0; k < iters; ++k) c->h_cnt[(size_t)k * NCOUNT + C_FLOPS] = h[(size_t)k];
  }
  if (c->profile) {
    auto span = [&](int k, int a, int b) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->pev[(size_t)k * kPev + a], c->pev[(size_t)k * kPev + b]);
      return ms;
    };
    c->first_ms = span(1, 6, 7);
    for (int k = 2; k <= iters; ++k) {
      const float hk = span(k, 0, 1);
      if (c->h_mode[k] == 0) {
        c->hook_ms += hk;
        ++c->hook_launches;
      } else {
        c->push_ms += hk;
      }
      if (c->HT && !FSV_FUSE_HUBFIX) c->hubfix_ms += span(k, 2, 3);
      if (c->comm && c->n) c->allreduce_ms += span(k, 8, 9);
      c->shortcut_ms += span(k, 6, 7);
    }
  }
  for (int k = 0; k < iters; ++k)
    if (c->h_cnt[(size_t)k * NCOUNT + C_VIOL])
      return fail(FSV_ERR_INVARIANT, "parent vector increased during kernel iteration");
  if (c->h_cnt[(size_t)(iters - 1) * NCOUNT + C_NONSTAR])
    return fail(FSV_ERR_INVARIANT, "algorithm terminated on non-star forest");
  return FSV_OK;
}

static void fill_stats(fsv_ctx* c, fsv_stats* s) {
  if (!s) return;
  memset(s, 0, sizeof *s);
  s->iterations = c->iterations;
  s->component_count = c->components;
  s->n = c->n;
  s->m_dir = c->m_dir;
  s->oriented_entries = c->E - c->R;  // edges only (headers excluded)
  s->hub_slots = c->HT;
  s->host_syncs = c->host_syncs;
  s->kernel_launches = c->launches;
  s->solve_ms = c->solve_ms;
  s->hook_ms = c->hook_ms;
  s->hubfix_ms = c->hubfix_ms;
  s->shortcut_ms = c->shortcut_ms;
  s->first_ms = c->first_ms;
  s->allreduce_ms = c->allreduce_ms;
  s->push_ms = c->push_ms;
  s->hook_launches = c->hook_launches;
  int sp = 0;
  for (int k = 2; k <= c->iterations && k < (int)c->h_mode.size(); ++k) sp += c->h_mode[k] == 1;
  s->sparse_iterations = sp;
  int mi = 0;
  for (int k = 0; k < c->iterations && (size_t)(k + 1) * NCOUNT <= c->h_cnt.size(); ++k)
    mi += c->h_cnt[(size_t)k * NCOUNT + C_MDONE] != 0;
  s->minority_iterations = mi;
  s->dense_exchanges = c->dense_x;
  s->delta_exchanges = c->delta_x;
  s->exchange_bytes = c->xbytes;
}

extern "C" int fsv_get_stats(fsv_ctx* c, fsv_stats* stats) {
  if (!c || !stats) return fail(FSV_ERR_CONTRACT, "NULL argument");
  fill_stats(c, stats);
  return FSV_OK;
}

extern "C" int fsv_solve(fsv_ctx* c, const fsv_config* cfg, fsv_stats* stats) {
  int rc = solve_impl(c, cfg, nullptr, 0);
  if (c) fill_stats(c, stats);
  return rc;
}

// ---- Labeling on the device (labeling_from_parents, graph.py:109-125) -----
// The star check and the component count come from the last vertex pass
// (C_NONSTAR, C_ROOTS). Sizes: warp-aggregated counts per representative
// (the giant component of a skewed graph would otherwise serialise one
// counter), then the representatives (label[u] == u, ascending) compacted
// with their sizes, and the labels widened to int64 (the reference's ID_DTYPE).
// Two levels of aggregation: lanes with the same label (match_any), then a
// per-block shared-memory table of labels (open addressing, flushed once per
// block), so the giant component of a skewed graph costs one global atomic
// per block instead of one per warp (all on one L2 line: 131 K for RMAT-22,
// 180 µs serialised). Labels that do not find a table slot go to global.
constexpr int kSizeSlots = 1024;   // power of two
__global__ void __launch_bounds__(256) k_comp_sizes(const int* __restrict__ L, long long n, unsigned* __restrict__ cnt) {
  __shared__ int s_key[kSizeSlots];
  __shared__ unsigned s_val[kSizeSlots];
  for (int i = threadIdx.x; i < kSizeSlots; i += blockDim.x) {
    s_key[i] = -1;
    s_val[i] = 0u;
  }
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += stride) {  // block-uniform
    const long long u = base + threadIdx.x;
    const bool on = u < n;
    const int l = on ? __ldg(L + u) : -1;
    const unsigned active = __ballot_sync(0xffffffffu, on);
    if (on) {
      const unsigned peers = __match_any_sync(active, l);
      if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) {
        const unsigned k = (unsigned)__popc(peers);
        unsigned h = ((unsigned)l * 2654435761u) >> 22;   // 10 bits
        bool done = k == 1u;   // a label alone in its warp: straight to global
        if (done) atomicAdd(cnt + l, 1u);
        for (int probe = 0; probe < 8 && !done; ++probe, h = (h + 1) & (kSizeSlots - 1)) {
          const int prev = atomicCAS(&s_key[h], -1, l);
          if (prev == -1 || prev == l) {
            atomicAdd(&s_val[h], k);
            done = true;
          }
        }
        if (!done) atomicAdd(cnt + l, k);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kSizeSlots; i += blockDim.x)
    if (s_key[i] >= 0) atomicAdd(cnt + s_key[i], s_val[i]);
}

struct IsRoot {
  const int* L;
  __device__ __forceinline__ bool operator()(int u) const { return __ldg(L + u) == u; }
};

__global__ void k_comp_out(const int* __restrict__ reps32, const int* __restrict__ num, const unsigned* __restrict__ cnt,
                           int64_t* __restrict__ reps, int64_t* __restrict__ sizes) {
  const long long C = *num;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < C; i += (long long)gridDim.x * blockDim.x) {
    const int r = reps32[i];
    reps[i] = r;
    sizes[i] = cnt[r];
  }
}

__global__ void k_widen(const int* __restrict__ in, long long n, int64_t* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = in[i];
}

static int build_labeling(fsv_ctx* c) {
  if (c->labeling_ready) return FSV_OK;
  const long long n = c->n;
  cudaStream_t st = c->stream;
  const int* L = c->labels_src ? c->labels_src : c->G;
  CUDA_TRY(c->lab.cnt.alloc((size_t)std::max<long long>(n, 1)));
  CUDA_TRY(c->lab.reps32.alloc((size_t)std::max<long long>(n, 1) + 1));   // + selected count
  CUDA_TRY(c->lab.reps.alloc((size_t)std::max<long long>(n, 1)));
  CUDA_TRY(c->lab.sizes.alloc((size_t)std::max<long long>(n, 1)));
  CUDA_TRY(c->lab.labels.alloc((size_t)std::max<long long>(n, 1)));
  int* d_num = c->lab.reps32.p + std::max<long long>(n, 1);
  CUDA_TRY(cudaMemsetAsync(c->lab.cnt.p, 0, sizeof(unsigned) * (size_t)std::max<long long>(n, 1), st));
  CUDA_TRY(cudaMemsetAsync(d_num, 0, sizeof(int), st));
  if (n) {
    k_comp_sizes<<<grid_for(c, n, 256), 256, 0, st>>>(L, n, c->lab.cnt.p);
    size_t bytes = 0;
    thrust::counting_iterator<int> ids(0);
    CUDA_TRY(cub::DeviceSelect::If(nullptr, bytes, ids, c->lab.reps32.p, d_num, (int)n, IsRoot{L}, st));
    CUDA_TRY(c->lab.tmp.alloc(std::max<size_t>(bytes, 1)));
    CUDA_TRY(cub::DeviceSelect::If(c->lab.tmp.p, bytes, ids, c->lab.reps32.p, d_num, (int)n, IsRoot{L}, st));
    k_comp_out<<<grid_for(c, n, 256), 256, 0, st>>>(c->lab.reps32.p, d_num, c->lab.cnt.p, c->lab.reps.p,
                                                     c->lab.sizes.p);
    k_widen<<<grid_for(c, n, 256), 256, 0, st>>>(L, n, c->lab.labels.p);
  }
  int num = 0;
  CUDA_TRY(cudaMemcpyAsync(&num, d_num, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  c->lab.count = num;
  c->labeling_ready = true;
  return FSV_OK;
}

extern "C" int fsv_get_labeling(fsv_ctx* c, int64_t* labels, int64_t* reps, int64_t* sizes, int64_t cap,
                                int64_t* count) {
  if (!c || !c->labels_ready) return fail(FSV_ERR_CONTRACT, "no solve result available");
  CUDA_TRY(cudaSetDevice(c->device));
  int rc = build_labeling(c);
  if (rc) return rc;
  const long long C = c->lab.count;
  if (count) *count = C;
  if ((reps || sizes) && cap < C)
    return fail(FSV_ERR_CONTRACT, "capacity %lld < %lld components", (long long)cap, C);
  if (labels && c->n && (rc = copy_out(c, labels, c->lab.labels.p, sizeof(int64_t) * c->n))) return rc;
  if (reps && C && (rc = copy_out(c, reps, c->lab.reps.p, sizeof(int64_t) * C))) return rc;
  if (sizes && C && (rc = copy_out(c, sizes, c->lab.sizes.p, sizeof(int64_t) * C))) return rc;
  return FSV_OK;
}

// Emulated rank group (tests): `count` contexts on one device, each holding
// one row range of the same graph, solved in lockstep with a device min-merge
// in place of the allreduce; see include/fastsv.h.
extern "C" int fsv_group_solve(fsv_ctx* const* ctxs, int count, const fsv_config* cfg, fsv_stats* stats) {
  if (!ctxs) return fail(FSV_ERR_CONTRACT, "NULL context array");
  int rc = solve_impl_group(ctxs, count, cfg, nullptr, 0);
  if (ctxs[0] && count >= 1) fill_stats(ctxs[0], stats);
  return rc;
}

extern "C" int fsv_group_run_snapshots(fsv_ctx* const* ctxs, int count, const fsv_config* cfg, int32_t* labels,
                                       int32_t* iterations, int64_t* gfc, int64_t* fc, int32_t* snapshots,
                                       int32_t snap_cap) {
  if (!ctxs) return fail(FSV_ERR_CONTRACT, "NULL context array");
  if (!snapshots) return fail(FSV_ERR_CONTRACT, "snapshots is NULL");
  int rc = solve_impl_group(ctxs, count, cfg, snapshots, snap_cap);
  fsv_ctx* c = ctxs[0];
  if (c && c->labels_ready) {
    if (iterations) *iterations = c->iterations;
    fsv_get_trace(c, gfc, fc, nullptr, snap_cap);
  }
  if (rc) return rc;
  return labels ? fsv_get_labels(c, labels) : FSV_OK;
}

extern "C" int fsv_get_labels(fsv_ctx* c, int32_t* labels) {
  if (!c || !c->labels_ready) return fail(FSV_ERR_CONTRACT, "no solve result available");
  if (!c->n) return FSV_OK;
  if (!labels) return fail(FSV_ERR_CONTRACT, "labels is NULL");
  CUDA_TRY(cudaSetDevice(c->device));
  return copy_out(c, labels, c->labels_src ? c->labels_src : c->G, sizeof(int) * c->n);
}

extern "C" int fsv_get_labels64(fsv_ctx* c, int64_t* labels) {
  if (!c || !c->labels_ready) return fail(FSV_ERR_CONTRACT, "no solve result available");
  if (!c->n) return FSV_OK;
  if (!labels) return fail(FSV_ERR_CONTRACT, "labels is NULL");
  std::vector<int32_t> tmp((size_t)c->n);
  int rc = fsv_get_labels(c, tmp.data());
  if (rc) return rc;
  for (int64_t i = 0; i < c->n; ++i) labels[i] = tmp[(size_t)i];
  return FSV_OK;
}

extern "C" int fsv_get_trace(fsv_ctx* c, int64_t* gfc, int64_t* fc, float* ms, int32_t cap) {
  if (!c || !c->labels_ready) return fail(FSV_ERR_CONTRACT, "no solve result available");
  const int k = std::min(cap, c->iterations);
  for (int i = 0; i < k; ++i) {
    if (gfc) gfc[i] = (int64_t)c->h_cnt[(size_t)i * NCOUNT + C_GF];
    if (fc) fc[i] = (int64_t)c->h_cnt[(size_t)i * NCOUNT + C_F];
    if (ms) ms[i] = c->iter_ms[(size_t)i];
  }
  return FSV_OK;
}

extern "C" int fsv_get_trace_ex(fsv_ctx* c, int64_t* gfc, int64_t* fc, float* ms, int32_t* kernel,
                                int64_t* flops, int32_t cap) {
  int rc = fsv_get_trace(c, gfc, fc, ms, cap);
  if (rc) return rc;
  const int k = std::min(cap, c->iterations);
  for (int i = 0; i < k; ++i) {
    const int md = (i + 1 < (int)c->h_mode.size()) ? c->h_mode[(size_t)i + 1] : 0;
    if (kernel) kernel[i] = c->variant ? 2 : md;   // 2: "none" (vertex-level fastsv trace)
    if (c->variant) {
      if (flops) flops[i] = 0;
      continue;
    }
    if (flops) {
      // dense product: m_dir (kernels.py:67-68); sparse: pushed degree sum
      // (kernels.py:94,102); iteration 1 sparse pushes the whole vector = m_dir
      flops[i] = (md == 1 && i > 0) ? (int64_t)c->h_cnt[(size_t)i * NCOUNT + C_FLOPS] : c->m_dir;
    }
  }
  return FSV_OK;
}

extern "C" int fsv_run(fsv_ctx* c, const fsv_config* cfg, int32_t* labels, int32_t* iterations,
                       int64_t* gfc, int64_t* fc, int32_t cap) {
  int rc = solve_impl(c, cfg, nullptr, 0);
  if (c && c->labels_ready) {
    if (iterations) *iterations = c->iterations;
    fsv_get_trace(c, gfc, fc, nullptr, cap);
  }
  if (rc) return rc;
  return labels ? fsv_get_labels(c, labels) : FSV_OK;
}

extern "C" int fsv_run_snapshots(fsv_ctx* c, const fsv_config* cfg, int32_t* labels,
                                 int32_t* iterations, int64_t* gfc, int64_t* fc,
                                 int32_t* snapshots, int32_t snap_cap) {
  if (!snapshots) return fail(FSV_ERR_CONTRACT, "snapshots is NULL");
  int rc = solve_impl(c, cfg, snapshots, snap_cap);
  if (c && c->labels_ready) {
    if (iterations) *iterations = c->iterations;
    fsv_get_trace(c, gfc, fc, nullptr, snap_cap);
  }
  if (rc) return rc;
  return labels ? fsv_get_labels(c, labels) : FSV_OK;
}

// ---------------------------------------------------------------------------
// multi-GPU

extern "C" int fsv_nccl_unique_id(void* id128) {
  if (!id128) return fail(FSV_ERR_CONTRACT, "id buffer is NULL");
  int rc = nccl_load();
  if (rc) return rc;
  ncclUniqueId id;
  NCCL_TRY(g_nccl.GetUniqueId(&id));
  memcpy(id128, &id, sizeof id);
  return FSV_OK;
}

extern "C" int fsv_nccl_attach(fsv_ctx* c, const void* id128, int nranks, int rank) {
  if (!c || !id128) return fail(FSV_ERR_CONTRACT, "NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(FSV_ERR_CONTRACT, "rank %d / nranks %d invalid", rank, nranks);
  int rc = nccl_load();
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(c->device));
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  if (c->comm) g_nccl.CommDestroy(c->comm);
  c->comm = nullptr;
  NCCL_TRY(g_nccl.CommInitRank(&c->comm, nranks, id, rank));
  c->nranks = nranks;
  c->rank = rank;
  return FSV_OK;
}

#ifdef FSV_DEBUG_TIMING
extern "C" int fsv_debug_timing(unsigned long long* out, int count) {
  CUDA_TRY(cudaMemcpyFromSymbol(out, fsv::g_dbg_t, sizeof(unsigned long long) * count));
  return FSV_OK;
}
#endif
