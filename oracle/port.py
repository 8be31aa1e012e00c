"""numpy restatement of the reference CPU hot path — TEST / BASELINE ONLY.

This is the ``cpu_baseline`` / ``bench.py --impl reference`` arm: the
reference package ``svcc`` is pure Python + numpy and cannot travel to the
GPU box (it lives under /root/reference), so its ``fastsv_la`` loop is
restated here with the same numpy primitives and the same work per
iteration, so that timing it on the box's host cores measures what the
reference would cost there:

  dense product   gather + np.minimum.reduceat over non-empty rows, rows split
                  into `workers` contiguous spans on a thread pool
                  (kernels.py:32-68)
  sparse product  push over the changed gf entries with chunked
                  np.minimum.at (kernels.py:71-102), chosen per iteration by
                  the strict-threshold rule (driver.py:51-61, 85-93, 115-116)
  hooks/shortcut  np.minimum.at through the index snapshot, two element-wise
                  mins, monotonicity check (kernels.py:110-127, driver.py:95-100)
  termination     gf = f[f]; stop when count(dup != gf) == 0 (driver.py:102-117)

Outputs (labels, iteration count, gf_changed trace) are checked against the
reference's golden vectors in tests/test_oracle.py.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

_SCATTER_CHUNK = 1 << 20


class PortGraph:
    """CSR with int64 arrays, as the reference's CsrGraph holds them."""

    def __init__(self, n, offsets, cols):
        self.n = int(n)
        self.offsets = np.asarray(offsets, dtype=np.int64)
        self.cols = np.asarray(cols, dtype=np.int64)
        self.deg = np.diff(self.offsets)

    @property
    def m(self):
        return int(self.cols.size)


def _pull_span(g: PortGraph, x, y, lo, hi):
    off = g.offsets[lo:hi + 1]
    first, last = off[0], off[-1]
    if first == last:
        return
    gathered = x[g.cols[first:last]]
    live = off[1:] > off[:-1]
    seg = np.minimum.reduceat(gathered, (off[:-1] - first)[live])
    part = y[lo:hi]
    part[live] = np.minimum(part[live], seg)


def pull_min(g: PortGraph, x, y, pool=None, workers=1):
    """y[u] <- min(y[u], min over N(u) of x) for non-empty rows."""
    if g.n == 0:
        return g.m
    cuts = np.linspace(0, g.n, workers + 1, dtype=np.int64)
    spans = [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:]) if a < b]
    if pool is not None and len(spans) > 1:
        list(pool.map(lambda s: _pull_span(g, x, y, *s), spans))
    else:
        for a, b in spans:
            _pull_span(g, x, y, a, b)
    return g.m


def push_min(g: PortGraph, idx, vals, y):
    """y[v] <- min over delta entries (u, val) with v in N(u)."""
    work = 0
    for s in range(0, idx.size, _SCATTER_CHUNK):
        part = idx[s:s + _SCATTER_CHUNK]
        pv = vals[s:s + _SCATTER_CHUNK]
        lens = g.deg[part]
        total = int(lens.sum())
        work += total
        if not total:
            continue
        starts = np.repeat(g.offsets[part], lens)
        ramp = np.arange(total, dtype=np.int64) - np.repeat(np.cumsum(lens) - lens, lens)
        np.minimum.at(y, g.cols[starts + ramp], np.repeat(pv, lens))
    return work


def fastsv_la(g: PortGraph, threshold=0.1, workers=1, mode="auto"):
    """Returns (labels int64, iterations, gf_changed list, kernels list)."""
    n = g.n
    f = np.arange(n, dtype=np.int64)
    gf = f.copy()
    prev_gf = f.copy()
    acc = f.copy()        # persistent mngf accumulator
    snap_idx = f.copy()   # f committed by the previous iteration
    pool = ThreadPoolExecutor(max_workers=workers) if workers > 1 else None
    gfc_trace, kinds = [], []
    use_sparse = mode == "sparse_only"
    delta = None
    try:
        while True:
            if use_sparse:
                if delta is None:
                    delta = (np.arange(n, dtype=np.int64), gf.copy())
                push_min(g, delta[0], delta[1], acc)
                kinds.append("sparse")
            else:
                pull_min(g, gf, acc, pool, workers)
                kinds.append("dense")
            before = f.copy()
            np.minimum.at(f, snap_idx, acc)
            np.minimum(f, acc, out=f)
            np.minimum(f, gf, out=f)
            if n and np.any(f > before):
                raise AssertionError("parent vector increased")
            snap_idx = f.copy()
            gf = f[f]
            changed = gf != prev_gf
            gfc = int(np.count_nonzero(changed))
            gfc_trace.append(gfc)
            if gfc == 0:
                break
            if mode == "dense_only":
                use_sparse = False
            elif mode == "sparse_only":
                use_sparse = True
            else:
                use_sparse = gfc < threshold * n
            delta = None
            if use_sparse:
                where = np.nonzero(changed)[0]
                delta = (where, gf[where].copy())
            prev_gf = gf.copy()
    finally:
        if pool is not None:
            pool.shutdown()
    return f, len(gfc_trace), gfc_trace, kinds
