// FastSV device kernels for sm_100a (B200). Integer, HBM/L2-bound, no tensor
// cores: nothing on this path is a dense contraction.
//
// One FastSV iteration k (all flags; algorithms.py:79-91 == driver.py:81-117)
// maps onto three launches over buffers F = f_k, G = gf_k, N = f_{k+1}
// (pre-initialised to gf_k, which folds the shortcut f <-min gf, E1):
//
//   k_hook      edge-parallel over the oriented layout (each undirected edge
//               stored once, in the row of its lower-(degree,id) endpoint):
//               row side   mngf run-min -> N[u], N[F[u]]  (aggressive/stochastic)
//               column side gf[u]       -> N[v], N[F[v]]  (same rules, v <- u)
//               gf of the top-H degree vertices ("hubs") is read from shared
//               memory; column-side writes aimed at hubs are min-reduced into
//               a compact hub accumulator instead of random N atomics.
//   k_hubfix    applies the hub accumulator (hub_acc[slot] -> N[h], N[F[h]]).
//   k_shortcut  vertex-parallel: gf_{k+1} = N[N], change counters, star and
//               monotonicity checks, next N init, hub gf refresh, and the
//               device-side convergence flag (last-block ticket).
//
// Iteration 1 is closed-form (F = G = id): f_1[u] = min(u, min neighbour id),
// precomputed at upload from the sorted CSR rows, so k_first does iteration 1
// including its shortcut phase in one vertex-parallel pass.
//
// All writes into N are filtered min-atomics; a write that cannot lower N is
// skipped using the read-only gf_k (N[x] <= gf_k[x] always, and
// gf_k[F[x]] <= gf_k[x], so val >= gf_k[x] makes both hooks no-ops).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fsv {

constexpr int INF = 0x7fffffff;
// Oriented layout entry codes (uint32):
//   header  HDR | u          first entry of the row of vertex u
//   edge    [HUB] | v/slot   neighbour v (or its hub slot) of the current row
constexpr uint32_t HDR = 0x80000000u;
constexpr uint32_t HUB = 0x40000000u;    // edge column is a hub: low bits = slot
constexpr uint32_t IDMASK = 0x3fffffffu;
constexpr int EPL = 8;                   // contiguous entries per lane per step
constexpr int STEP = 32 * EPL;           // entries per warp step
constexpr int STEPS = 4;                 // steps per span
constexpr int SPAN = STEP * STEPS;       // entries per warp task
constexpr int HOOK_THREADS = 768;
constexpr int SC_THREADS = 512;
constexpr int NCOUNT = 8;                // counters per iteration
enum { C_GF = 0, C_F = 1, C_NONSTAR = 2, C_ROOTS = 3, C_VIOL = 4 };

// ---- memory helpers -------------------------------------------------------

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Streamed once per iteration: evict first from L2 so the parent vectors
// stay L2-resident. L1 may allocate: a lane's two 16-byte halves share sectors.
__device__ __forceinline__ uint4 ld_stream(const uint4* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ int ldg(const int* p) { return __ldg(p); }

__device__ __forceinline__ void red_min(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.min.s32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// ---- argument blocks --------------------------------------------------------

struct HookArgs {
  const uint32_t* ecol;   // oriented entries (headers + edges), padded to SPAN
  long long nspans;
  const int* span_row;    // vertex of the row open at each span start, -1 if none
  const int* F;           // f_k
  const int* G;           // gf_k
  int* N;                 // f_{k+1}, pre-initialised to gf_k
  const int* G_hub;       // gf_k of hub slots (compact)
  int H;                  // hub slots (multiple of 4)
  int* hub_acc;           // column-side minima aimed at hubs
  const int* done;        // convergence flag (iteration number, 0 = running)
};

struct ShortcutArgs {
  int* F;                 // in: f_k; out: gf_{k+1} (next N init)
  int* G;                 // in: gf_k; out: gf_{k+1}
  const int* N;           // f_{k+1}
  long long n;
  const int* hub_id;
  int* G_hub;
  int H;
  unsigned long long* cnt;  // this iteration's NCOUNT counters
  unsigned* partials;       // per-block partial counters [grid][8]
  unsigned int* ticket;
  int* done;
  int iter;               // 1-based iteration number
  int max_iter;           // stop flag raised when reached without converging
};

// ---- emission of one hook contribution -------------------------------------

// Row side: run minimum `val` of row vertex u (gu = gf_k[u]).
__device__ __forceinline__ void emit_row(int u, int gu, int val, const int* __restrict__ F,
                                         const int* __restrict__ G, int* __restrict__ N) {
  if (val < gu) {
    red_min(N + u, val);                 // aggressive: f[u] <-min mngf[u]
    int t = ldg(F + u);
    if (t != u && val < ldg(G + t)) red_min(N + t, val);  // stochastic: f[f[u]] <-min mngf[u]
  }
}

// Column side of edge entry c of a row whose gf is gu: v <- gu (kept for
// the hub-accumulator fix-up path and for clarity; k_hook batches these).
__device__ __forceinline__ void emit_col(uint32_t c, int gu, const int* __restrict__ F,
                                         const int* __restrict__ G, int* __restrict__ N,
                                         int* __restrict__ hub_acc) {
  const int x = (int)(c & IDMASK);
  if (c & HUB) {
    red_min(hub_acc + x, gu);
  } else {
    red_min(N + x, gu);
    int t = ldg(F + x);
    if (t != x && gu < ldg(G + t)) red_min(N + t, gu);
  }
}

// One gathered gf value per entry: hub edges from the shared-memory table
// (32-bit shared address, no generic conversion), everything else from
// global through the read-only path. Both loads are predicated, no branch.
__device__ __forceinline__ int gather_gf(uint32_t c, uint32_t s_base, const int* __restrict__ G) {
  int v;
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "@p  ld.shared.b32 %0, [%2];\n\t"
      "@!p ld.global.nc.b32 %0, [%3];\n\t}"
      : "=r"(v)
      : "r"(c & HUB), "r"(s_base + (c << 2)), "l"(G + (c & IDMASK)));
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

__global__ void __launch_bounds__(HOOK_THREADS, 1) k_hook(HookArgs a) {
  extern __shared__ int s_hub[];
  if (*(volatile const int*)a.done) return;
  for (int i = threadIdx.x; i < (a.H >> 2); i += blockDim.x)
    reinterpret_cast<int4*>(s_hub)[i] = reinterpret_cast<const int4*>(a.G_hub)[i];
  __syncthreads();
  const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(s_hub);

  const int* __restrict__ F = a.F;
  const int* __restrict__ G = a.G;
  int* __restrict__ N = a.N;
  int* __restrict__ hub_acc = a.hub_acc;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint64_t pol = policy_evict_first();

  for (long long s = gw; s < a.nspans; s += nwarps) {
    int carry_u = ldg(a.span_row + s);              // row open at the span start
    int carry_gu = carry_u >= 0 ? ldg(G + carry_u) : INF;
    int carry_run = INF;
    const uint4* p = reinterpret_cast<const uint4*>(a.ecol + s * SPAN) + 2 * lane;
    uint4 n0 = ld_stream(p, pol), n1 = ld_stream(p + 1, pol);
#pragma unroll 1
    for (int st = 0; st < STEPS; ++st) {
      const uint32_t c[EPL] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
      if (st + 1 < STEPS) {
        n0 = ld_stream(p + (st + 1) * 64, pol);
        n1 = ld_stream(p + (st + 1) * 64 + 1, pol);
      }
      int val[EPL];
#pragma unroll
      for (int j = 0; j < EPL; ++j) val[j] = gather_gf(c[j], s_base, G);
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
      // does any entry differ from its row's gf?
      bool need = false;
      {
        int rg = in_gu;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          rg = ((int)c[j] < 0) ? val[j] : rg;
          need |= (val[j] != rg);
        }
      }
      if (!__any_sync(0xffffffffu, need) && carry_run >= carry_gu) {
        if (hb) {
          const int last = 31 - __clz(hb);
          carry_u = __shfl_sync(0xffffffffu, lu, last);
          carry_gu = __shfl_sync(0xffffffffu, lgu, last);
          carry_run = INF;
        }
        continue;
      }
      // ---- slow path ------------------------------------------------------
      // One emission slot per entry, filled branch-free:
      //   header j: closes the row before it (the lane's first header closes
      //             the row entering the lane; handled after the scan)
      //             target = previous row vertex, value = its run min,
      //             threshold = its gf
      //   edge j:   column side, target = v (or hub slot), value = row gf,
      //             threshold = gf[v]
      // then every active slot does N[target] <-min value and the stochastic
      // N[F[target]] <-min value, with all loads of the lane in flight together.
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
        hubm |= (!h && (c[j] & HUB) ? 1u : 0u) << j;
        seen |= h;
        cu = h ? (int)(c[j] & IDMASK) : cu;
        cgu = h ? val[j] : cgu;
        run = h ? INF : min(run, val[j]);
      }
      if (act) {
        int t[EPL];
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          t[j] = -1;
          if ((act >> j) & 1u) {
            if ((hubm >> j) & 1u) {
              red_min(hub_acc + w[j], y[j]);
            } else {
              red_min(N + w[j], y[j]);
              t[j] = ldg(F + w[j]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          if (t[j] == w[j]) t[j] = -1;
          if (t[j] >= 0) val[j] = ldg(G + t[j]);
        }
#pragma unroll
        for (int j = 0; j < EPL; ++j)
          if (t[j] >= 0 && y[j] < val[j]) red_min(N + t[j], y[j]);
      }
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
        if (v < in_gu) emit_row(in_u, in_gu, v, F, G, N);  // row entering the lane closes here
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
    if (lane == 0 && carry_run < carry_gu) emit_row(carry_u, carry_gu, carry_run, F, G, N);
  }
}

// ---- hub accumulator -> N ---------------------------------------------------

__global__ void k_hubfix(int* __restrict__ hub_acc, const int* __restrict__ hub_id, int H,
                         const int* __restrict__ F, const int* __restrict__ G, int* __restrict__ N,
                         const int* done) {
  if (*(volatile const int*)done) return;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < H; s += gridDim.x * blockDim.x) {
    const int acc = hub_acc[s];
    if (acc == INF) continue;
    hub_acc[s] = INF;
    const int h = ldg(hub_id + s);
    emit_row(h, ldg(G + h), acc, F, G, N);
  }
}

// ---- counters + convergence flag --------------------------------------------
// Each block writes its five partial counts; the last block to finish (ticket)
// sums them, stores this iteration's counters and raises the convergence flag
// when gf did not change. No same-address atomics besides the ticket.

template <int NT>
__device__ __forceinline__ void finish_counters(const unsigned (&c)[5], unsigned* partials,
                                                unsigned long long* cnt, unsigned int* ticket,
                                                int* done, int iter, int max_iter) {
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
  if (threadIdx.x < 5) {
    unsigned long long sum = 0;
    for (int i = 0; i < NT / 32; ++i) sum += s_acc[i][threadIdx.x];
    cnt[threadIdx.x] = sum;
    if (threadIdx.x == C_GF) {
      if (sum == 0ull) atomicExch(done, iter);
      else if (max_iter > 0 && iter >= max_iter) atomicExch(done, -iter);
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// ---- phase G: grandparents, counters, next N init ---------------------------

__device__ __forceinline__ void shortcut_group(long long i, const int4* N4, const int* __restrict__ N,
                                               int4* F4, int4* G4, unsigned (&c)[5]) {
  const int4 nu = N4[i];
  const int4 go = G4[i];
  const int4 fo = F4[i];
  int4 gg;
  gg.x = ldg(N + nu.x); gg.y = ldg(N + nu.y); gg.z = ldg(N + nu.z); gg.w = ldg(N + nu.w);
  const int u = (int)(i << 2);
  c[C_GF] += (gg.x != go.x) + (gg.y != go.y) + (gg.z != go.z) + (gg.w != go.w);
  c[C_F] += (nu.x != fo.x) + (nu.y != fo.y) + (nu.z != fo.z) + (nu.w != fo.w);
  c[C_NONSTAR] += (gg.x != nu.x) + (gg.y != nu.y) + (gg.z != nu.z) + (gg.w != nu.w);
  c[C_ROOTS] += (nu.x == u) + (nu.y == u + 1) + (nu.z == u + 2) + (nu.w == u + 3);
  c[C_VIOL] += (nu.x > fo.x) + (nu.y > fo.y) + (nu.z > fo.z) + (nu.w > fo.w);
  G4[i] = gg;
  F4[i] = gg;
}

__global__ void __launch_bounds__(SC_THREADS) k_shortcut(ShortcutArgs a) {
  if (*(volatile const int*)a.done) return;
  unsigned c[5] = {0u, 0u, 0u, 0u, 0u};
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n4 = a.n >> 2;
  const int* __restrict__ N = a.N;
  int4* F4 = reinterpret_cast<int4*>(a.F);
  int4* G4 = reinterpret_cast<int4*>(a.G);
  const int4* N4 = reinterpret_cast<const int4*>(a.N);
  long long i = t0;
  for (; i + stride < n4; i += 2 * stride) {   // two independent groups in flight
    shortcut_group(i, N4, N, F4, G4, c);
    shortcut_group(i + stride, N4, N, F4, G4, c);
  }
  if (i < n4) shortcut_group(i, N4, N, F4, G4, c);
  for (long long u = (n4 << 2) + t0; u < a.n; u += stride) {
    const int nu = N[u], go = a.G[u], fo = a.F[u];
    const int gg = ldg(N + nu);
    c[C_GF] += gg != go; c[C_F] += nu != fo; c[C_NONSTAR] += gg != nu;
    c[C_ROOTS] += nu == (int)u; c[C_VIOL] += nu > fo;
    a.G[u] = gg; a.F[u] = gg;
  }
  for (long long s = t0; s < a.H; s += stride) {
    const int h = ldg(a.hub_id + s);
    a.G_hub[s] = ldg(N + ldg(N + h));
  }
  finish_counters<SC_THREADS>(c, a.partials, a.cnt, a.ticket, a.done, a.iter, a.max_iter);
}

// ---- iteration 1 in closed form ---------------------------------------------
// f_1[u] = min(u, min neighbour) = f1[u]; gf_1 = f1[f1]. Writes Y = f_1,
// G = gf_1 and X = gf_1 (the N init of iteration 2).
__global__ void __launch_bounds__(SC_THREADS) k_first(const int* __restrict__ f1, int* Y, int* G,
                                                      int* X, long long n, const int* __restrict__ hub_id,
                                                      int* G_hub, int H, unsigned long long* cnt,
                                                      unsigned* partials, unsigned int* ticket,
                                                      int* done, int max_iter) {
  unsigned c[5] = {0u, 0u, 0u, 0u, 0u};
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n4 = n >> 2;
  const int4* f14 = reinterpret_cast<const int4*>(f1);
  for (long long i = t0; i < n4; i += stride) {
    const int4 a = f14[i];
    int4 gg;
    gg.x = ldg(f1 + a.x); gg.y = ldg(f1 + a.y); gg.z = ldg(f1 + a.z); gg.w = ldg(f1 + a.w);
    const int u = (int)(i << 2);
    c[C_GF] += (gg.x != u) + (gg.y != u + 1) + (gg.z != u + 2) + (gg.w != u + 3);
    c[C_F] += (a.x != u) + (a.y != u + 1) + (a.z != u + 2) + (a.w != u + 3);
    c[C_NONSTAR] += (gg.x != a.x) + (gg.y != a.y) + (gg.z != a.z) + (gg.w != a.w);
    c[C_ROOTS] += (a.x == u) + (a.y == u + 1) + (a.z == u + 2) + (a.w == u + 3);
    c[C_VIOL] += (a.x > u) + (a.y > u + 1) + (a.z > u + 2) + (a.w > u + 3);
    reinterpret_cast<int4*>(Y)[i] = a;
    reinterpret_cast<int4*>(G)[i] = gg;
    reinterpret_cast<int4*>(X)[i] = gg;
  }
  for (long long u = (n4 << 2) + t0; u < n; u += stride) {
    const int a = f1[u];
    const int gg = ldg(f1 + a);
    c[C_GF] += gg != (int)u; c[C_F] += a != (int)u; c[C_NONSTAR] += gg != a;
    c[C_ROOTS] += a == (int)u; c[C_VIOL] += a > (int)u;
    Y[u] = a; G[u] = gg; X[u] = gg;
  }
  for (long long s = t0; s < H; s += stride) {
    const int h = ldg(hub_id + s);
    G_hub[s] = ldg(f1 + ldg(f1 + h));
  }
  finish_counters<SC_THREADS>(c, partials, cnt, ticket, done, 1, max_iter);
}

// ---- solve-start initialisation ----------------------------------------------
__global__ void k_solve_init(int* X, int* Y, int* G, long long n, int* hub_acc, int H,
                             unsigned long long* cnt, long long ncnt, int* done, unsigned* ticket) {
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long s = t0; s < H; s += stride) hub_acc[s] = INF;
  for (long long k = t0; k < ncnt; k += stride) cnt[k] = 0ull;
  if (t0 == 0) {
    X[n] = (int)n; Y[n] = (int)n; G[n] = INF;  // dummy vertex n of the padding row
    *done = 0; *ticket = 0u;
  }
}

}  // namespace fsv
