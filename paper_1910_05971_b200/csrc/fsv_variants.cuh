// Weaker hooking variants of FastSV on the device: the reference's
// HookingConfig ablation (algorithms.py:28-35, _fastsv_iteration :79-100,
// stop rule _uses_gf_termination :103-114) and simplified_sv (:66-76,
// :145-149). Not the hot path (the all-flags algorithm runs on the oriented
// layout in fsv_kernels.cuh): these run edge-parallel over the resident
// symmetric CSR with a per-entry row id (CsrGraph.row_ids, graph.py:47-52),
// filtered min-reductions and vertex passes. Integer min is order
// independent, so every committed parent vector equals the reference's.
//
// One iteration, buffers F = f, G = gf = f[f] (read only), N = f_next:
//   stochastic on (one commit, algorithms.py:85-92):
//     N = min(f, gf)                         (the final min with gf, folded)
//     N[f[u]] <-min val, [aggressive] N[u] <-min val     for stored (u, v)
//   stochastic off (two commits, algorithms.py:93-100):
//     N = f;  N[f[u]] <-min val if gf[u] == f[u] (u's parent is a root),
//     [aggressive] N[u] <-min val;   T = min(N, N[N])   (shortcut on post-hook N)
//   val = gf[v] with grandparent hooking, f[v] without.
// A reduction into N[x] is skipped when val cannot lower N[x]'s start value.
#pragma once
#include <cstdint>

namespace fsv {

// Row id of every stored entry of rows [row_begin, row_end): a warp per row.
__global__ void k_row_ids(const int64_t* __restrict__ off, long long col_base, long long row_begin,
                          long long row_end, int* __restrict__ rows) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long r = row_begin + (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < row_end;
       r += nw) {
    const long long lo = off[r] - col_base, hi = off[r + 1] - col_base;
    for (long long e = lo + lane; e < hi; e += 32) rows[e] = (int)r;
  }
}

__global__ void k_var_iota(int* __restrict__ F, int* __restrict__ G, long long n) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n; u += (long long)gridDim.x * blockDim.x) {
    F[u] = (int)u;
    G[u] = (int)u;
  }
}

__global__ void k_var_init(const int* __restrict__ F, const int* __restrict__ G, int* __restrict__ N, long long n,
                           bool with_gf) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n; u += (long long)gridDim.x * blockDim.x)
    N[u] = with_gf ? min(F[u], G[u]) : F[u];
}

template <bool STO, bool AGG, bool GP>
__global__ void k_var_hook(const int* __restrict__ rows, const int* __restrict__ cols, long long m,
                           const int* __restrict__ F, const int* __restrict__ G, int* __restrict__ N) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m; e += (long long)gridDim.x * blockDim.x) {
    const int u = __ldg(rows + e), v = __ldg(cols + e);
    const int val = GP ? __ldg(G + v) : __ldg(F + v);
    const int fu = __ldg(F + u), gu = __ldg(G + u);
    // N[f[u]] starts at <= f[f[u]] = gf[u]; N[u] at <= f[u]
    if ((STO || gu == fu) && val < gu) red_min(N + fu, val);
    if (AGG && val < fu) red_min(N + u, val);
  }
}

// Adds this block's counts to cnt[0..NC) (one atomic per counter per block).
template <int NC>
__device__ __forceinline__ void block_count(const unsigned (&c)[NC], unsigned long long* cnt) {
  __shared__ unsigned s[32][NC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const unsigned v = __reduce_add_sync(0xffffffffu, c[k]);
    if (lane == 0) s[w][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < NC) {
    unsigned long long sum = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) sum += s[i][threadIdx.x];
    if (sum) atomicAdd(cnt + threadIdx.x, sum);
  }
}

// Two-commit variants: T = min(N, N[N]) (the shortcut reads post-hook parents).
__global__ void k_var_shortcut(const int* __restrict__ N, int* __restrict__ T, long long n) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n; u += (long long)gridDim.x * blockDim.x) {
    const int x = N[u];
    T[u] = min(x, __ldg(N + x));
  }
}

// Commit bookkeeping of the new parent vector P (= N or T): Gn = P[P] and the
// trace counters against the previous committed f (F) and gf (G):
// cnt[0] gf_changed, [1] f_changed, [2] non-star, [3] roots, [4] increases.
__global__ void k_var_count(const int* __restrict__ P, const int* __restrict__ F, const int* __restrict__ G,
                            int* __restrict__ Gn, long long n, unsigned long long* cnt) {
  unsigned c[5] = {0u, 0u, 0u, 0u, 0u};
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n; u += (long long)gridDim.x * blockDim.x) {
    const int p = P[u];
    const int g = __ldg(P + p);
    Gn[u] = g;
    c[0] += g != G[u];
    c[1] += p != F[u];
    c[2] += g != p;
    c[3] += p == (int)u;
    c[4] += p > F[u];
  }
  block_count<5>(c, cnt);
}

}  // namespace fsv
