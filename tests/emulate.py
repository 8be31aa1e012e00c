"""numpy emulation of the device schedule (test-only).

Mirrors what libfastsv.so does, step for step, so the host-side partition
logic and the collective semantics can be tested on CPU:

  layout     each undirected edge {a, b} kept once, in the row of the endpoint
             that comes later in the degree-descending order, ties by id
             (k_positions + k_orient_encode/k_orient_compact)
  iteration 1  f1[u] = min(u, smallest neighbour) from each rank's own rows,
             assembled with an allreduce-min (k_f1 + ncclAllReduce)
  iteration k>=2 on every rank, over its own oriented entries (k_hook):
             row side    run-min of gf over the row  -> N[u]
             column side gf[row]                     -> N[v]
             each filtered by "value < gf_k[target]" (aggressive hooks); then
             allreduce-min of N (ncclAllReduce ncclMin) and the replicated
             vertex pass (k_shortcut): the deferred stochastic hooks
             N[F[u]] <-min N[u] for every u the sweep lowered (N[u] < gf_k[u],
             all values read before any is lowered), then gf' = N[N] with the
             gf-stability stop rule. A sparse iteration (the library's push)
             applies both hooks per contribution instead (N[u] and N[F[u]]).

``allreduce_min`` is injected so the same code runs single-process (identity)
or across gloo ranks (torch.distributed.all_reduce with ReduceOp.MIN).

Sparse iterations (the reference's rule, gf_changed < 0.1 n, driver.py:51-61)
may instead take the library's delta exchange (fsv_config.exchange = 0): each
rank's (index, value) pairs of the entries it lowered (N[i] < gf_k[i]) are
all-gathered (``allgather_pairs``: counts first, then the lists padded to the
largest, as k_delta_compact + two ncclAllGathers) and min-reduced into N
(k_delta_apply), falling back to the allreduce when the lists are not smaller.
"""

from __future__ import annotations

import numpy as np

INF = np.iinfo(np.int32).max


def oriented_entries(n, offsets, cols, row_begin, row_end):
    """(rows, cols) of the oriented entries owned by rows [row_begin, row_end)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    deg = np.diff(offsets)
    lo, hi = offsets[row_begin], offsets[row_end]
    rows = np.repeat(np.arange(row_begin, row_end, dtype=np.int64), deg[row_begin:row_end])
    c = np.asarray(cols, dtype=np.int64)[lo:hi] if cols.size else np.zeros(0, np.int64)
    order = np.argsort(-deg, kind="stable")        # degree-descending, ties by id
    pos = np.empty(n, dtype=np.int64)
    pos[order] = np.arange(n)
    keep = pos[c] < pos[rows]
    return rows[keep], c[keep]


def first_parents(n, offsets, cols, row_begin, row_end):
    """Partial f1 (INF outside the rank's rows)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    f1 = np.full(n, INF, dtype=np.int64)
    u = np.arange(row_begin, row_end, dtype=np.int64)
    f1[u] = u
    nz = u[offsets[u + 1] > offsets[u]]
    if nz.size:
        f1[nz] = np.minimum(nz, np.asarray(cols, dtype=np.int64)[offsets[nz]])
    return f1


def _scatter_min(target, idx, vals):
    if idx.size:
        np.minimum.at(target, idx, vals)


def hook(rows, cols, F, G, N, stochastic=True):
    """One rank's phase H over its oriented entries (N modified in place).
    stochastic=False: aggressive hooks only (the dense sweep; the vertex pass
    then runs deferred_stochastic)."""
    if rows.size == 0:
        return
    gv = G[cols]
    gu = G[rows]
    # row side: per-row minimum of gv (rows are sorted)
    starts = np.flatnonzero(np.r_[True, rows[1:] != rows[:-1]])
    rmin = np.minimum.reduceat(gv, starts)
    ru = rows[starts]
    ok = rmin < G[ru]
    u, val = ru[ok], rmin[ok]
    _scatter_min(N, u, val)
    if stochastic:
        t = F[u]
        ok2 = (t != u) & (val < G[t])
        _scatter_min(N, t[ok2], val[ok2])
    # column side: v <- gf[row]
    ok = gu < gv
    v, val = cols[ok], gu[ok]
    _scatter_min(N, v, val)
    if stochastic:
        t = F[v]
        ok2 = (t != v) & (val < G[t])
        _scatter_min(N, t[ok2], val[ok2])


def deferred_stochastic(F, G, N):
    """The vertex pass's first step after a dense sweep (k_shortcut): every
    vertex the aggressive hooks lowered hooks its parent with its new value,
    all values read before any reduction lands."""
    u = np.flatnonzero(N < G)
    val = N[u].copy()
    t = F[u]
    ok = t != u
    _scatter_min(N, t[ok], val[ok])


def delta_exchange(N, G, allgather_pairs, nranks):
    """The sparse-iteration exchange; returns (N merged, bytes this rank sent)."""
    idx = np.flatnonzero(N < G)
    mine = np.stack([idx, N[idx]], 1).astype(np.int64)
    lists = allgather_pairs(mine)
    cmax = max(len(x) for x in lists)
    if 8 * cmax * nranks >= 2 * (nranks - 1) / nranks * 4 * N.size:
        return None, 0
    out = N.copy()
    for x in lists:
        if len(x):
            np.minimum.at(out, x[:, 0], x[:, 1])
    return out, 8 * cmax * (nranks - 1)


def run(n, offsets, cols, row_begin=0, row_end=None, allreduce_min=lambda a: a,
        cap=4096, record=True, allgather_pairs=None, nranks=1, stats=None, threshold=0.1):
    """Returns (labels, iterations, gf_changed, f_changed, snapshots). With
    ``allgather_pairs``, sparse iterations use the delta exchange; ``stats``
    (a dict) then receives the exchange counts and bytes."""
    row_end = n if row_end is None else row_end
    rows, ocols = oriented_entries(n, offsets, cols, row_begin, row_end)
    f1 = allreduce_min(first_parents(n, offsets, cols, row_begin, row_end))
    F = f1.copy()                        # f_1
    G = f1[f1]                           # gf_1
    ident = np.arange(n, dtype=np.int64)
    gfc = [int(np.count_nonzero(G != ident))]
    fc = [int(np.count_nonzero(F != ident))]
    snaps = [F.copy()] if record else None
    it = 1
    while gfc[-1] != 0 and it < cap:
        it += 1
        N = G.copy()                     # f_k initialised to gf_{k-1} (shortcut folded)
        sparse = gfc[-1] < threshold * n
        hook(rows, ocols, F, G, N, stochastic=sparse)
        merged = None
        if allgather_pairs is not None and sparse:
            merged, sent = delta_exchange(N, G, allgather_pairs, nranks)
        if merged is not None:
            N = merged
            if stats is not None:
                stats["delta"] = stats.get("delta", 0) + 1
                stats["bytes"] = stats.get("bytes", 0) + sent
        else:
            N = allreduce_min(N)
            if stats is not None:
                stats["dense"] = stats.get("dense", 0) + 1
        if not sparse:
            deferred_stochastic(F, G, N)
        G2 = N[N]
        gfc.append(int(np.count_nonzero(G2 != G)))
        fc.append(int(np.count_nonzero(N != F)))
        if np.any(N > F):
            raise AssertionError("parent increased")
        F, G = N, G2
        if record:
            snaps.append(F.copy())
    if n and not np.array_equal(F[F], F):
        raise AssertionError("non-star at exit")
    return F, it, gfc, fc, snaps
