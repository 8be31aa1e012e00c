"""Inputs of the reference arm, in pure numpy (no native library of this repo).

`bench.py --impl reference` must time the UNMODIFIED reference (`svcc`,
installed into baseline/_ref) on the same graph as our arm without mapping
any of this repo's shared objects into the reference process. This module
regenerates BASELINE.json's configs bit-identically to the repo's C++
generators (paper_1910_05971_b200/csrc/fsv_graphgen.cpp: Philox-4x32-10
keyed by (seed, stream, index), RMAT one 32-bit draw per level, Fisher-Yates
id permutation from the top) and builds the symmetric CSR with
svcc.build_csr's semantics (graph.py:55-97: self-loops dropped, both
orientations, duplicates merged, rows sorted) with a bucketed numpy sort
(svcc.build_csr itself takes minutes at RMAT-22; only its product matters
here, and tests/test_ref_inputs.py pins both to the repo's builder).

Host threads: numpy ufuncs release the GIL, so chunks run on a thread pool.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

U64 = np.uint64
MASK32 = U64(0xFFFFFFFF)
M0, M1 = U64(0xD2511F53), U64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
STREAM_RMAT, STREAM_PERM, STREAM_GRID = 1, 2, 3
STREAM_TREE_SIZE, STREAM_TREE_PARENT, STREAM_TREE_EXTRA = 4, 5, 6
RMAT_ABC = (0.57, 0.19, 0.19)


def threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def philox4x32(c0, c1, c2, c3, seed: int):
    """Philox-4x32-10 on uint64 arrays holding 32-bit lanes (csrc/philox.h)."""
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    c0 = np.asarray(c0, dtype=U64)
    c1 = np.asarray(c1, dtype=U64)
    c2 = np.asarray(c2, dtype=U64)
    c3 = np.asarray(c3, dtype=U64)
    for _ in range(10):
        p0 = c0 * M0
        p1 = c2 * M1
        n0 = (p1 >> U64(32)) ^ c1 ^ U64(k0)
        n2 = (p0 >> U64(32)) ^ c3 ^ U64(k1)
        c0, c1, c2, c3 = n0, p1 & MASK32, n2, p0 & MASK32
        k0 = (k0 + W0) & 0xFFFFFFFF
        k1 = (k1 + W1) & 0xFFFFFFFF
    return c0, c1, c2, c3


def draw4(seed: int, stream: int, index, group: int = 0):
    idx = np.asarray(index, dtype=U64)
    return philox4x32(idx & MASK32, idx >> U64(32), U64(group), U64(stream), seed)


def bounded(r, rng):
    """Lemire multiply-shift: uniform in [0, rng) from a 32-bit draw."""
    return (np.asarray(r, dtype=U64) * np.asarray(rng, dtype=U64)) >> U64(32)


def _parallel(fn, total: int, chunk: int = 1 << 21):
    with ThreadPoolExecutor(threads()) as ex:
        list(ex.map(lambda lo: fn(lo, min(total, lo + chunk)), range(0, total, chunk)))


def permutation(n: int, seed: int) -> np.ndarray:
    """Fisher-Yates from the top; position i swaps with j = floor(r64 * (i+1) / 2^64)."""
    perm = np.arange(n, dtype=np.int32)
    if n <= 1:
        return perm
    js = np.empty(n, dtype=np.int64)

    def fill(lo, hi):
        i = np.arange(lo, hi, dtype=U64)
        v0, v1, _, _ = draw4(seed, STREAM_PERM, i)
        t = i + U64(1)
        js[lo:hi] = ((v1 * t + ((v0 * t) >> U64(32))) >> U64(32)).astype(np.int64)

    _parallel(fill, n)
    p = perm.tolist()
    jl = js.tolist()
    for i in range(n - 1, 0, -1):
        j = jl[i]
        p[i], p[j] = p[j], p[i]
    return np.asarray(p, dtype=np.int32)


def rmat(scale: int, edgefactor: int = 16, abc=RMAT_ABC, seed: int = 0, permute: bool = True):
    n = 1 << scale
    m = edgefactor * n
    a, b, c = abc
    tA = U64(int(np.floor(a * 4294967296.0 + 0.5)))
    tAB = U64(int(np.floor((a + b) * 4294967296.0 + 0.5)))
    tABC = U64(int(np.floor((a + b + c) * 4294967296.0 + 0.5)))
    pairs = np.empty((m, 2), dtype=np.int32)
    groups = (scale + 3) // 4

    def fill(lo, hi):
        i = np.arange(lo, hi, dtype=U64)
        row = np.zeros(hi - lo, dtype=U64)
        col = np.zeros(hi - lo, dtype=U64)
        for g in range(groups):
            r = draw4(seed, STREAM_RMAT, i, g)
            for w in range(4):
                level = 4 * g + w
                if level >= scale:
                    break
                x = r[w]
                bit = U64(1 << (scale - 1 - level))
                col |= np.where(((x >= tA) & (x < tAB)) | (x >= tABC), bit, U64(0))
                row |= np.where(x >= tAB, bit, U64(0))
        pairs[lo:hi, 0] = row.astype(np.int32)
        pairs[lo:hi, 1] = col.astype(np.int32)

    _parallel(fill, m)
    if permute:
        pairs = permutation(n, seed)[pairs]
    return n, pairs


def grid(rows: int, cols: int, p_drop: float = 0.4, seed: int = 0, permute: bool = True):
    H = rows * (cols - 1)
    total = H + (rows - 1) * cols
    thr = U64(int(np.floor(p_drop * 4294967296.0 + 0.5)))
    e = np.arange(total, dtype=np.int64)
    keep = np.empty(total, dtype=bool)

    def fill(lo, hi):
        keep[lo:hi] = draw4(seed, STREAM_GRID, np.arange(lo, hi, dtype=U64))[0] >= thr

    _parallel(fill, total)
    e = e[keep]
    h = e < H
    u = np.where(h, (e // max(cols - 1, 1)) * cols + e % max(cols - 1, 1), e - H)
    v = np.where(h, u + 1, u + cols)
    pairs = np.stack([u, v], 1).astype(np.int32)
    if permute:
        pairs = permutation(rows * cols, seed)[pairs]
    return rows * cols, pairs


def forest(trees: int, min_size: int = 1, max_size: int = 64, extra: int = 2, seed: int = 0,
           permute: bool = True):
    span = max_size - min_size + 1
    t = np.arange(trees, dtype=U64)
    sizes = (min_size + bounded(draw4(seed, STREAM_TREE_SIZE, t)[0], span)).astype(np.int64)
    base = np.zeros(trees + 1, dtype=np.int64)
    np.cumsum(sizes, out=base[1:])
    epert = sizes - 1 + extra
    ebase = np.zeros(trees + 1, dtype=np.int64)
    np.cumsum(epert, out=ebase[1:])
    n, m = int(base[-1]), int(ebase[-1])
    pairs = np.empty((m, 2), dtype=np.int32)
    tree_of = np.repeat(np.arange(trees, dtype=np.int64), sizes)
    g = np.arange(n, dtype=np.int64)
    i = g - base[tree_of]
    nr = i > 0
    gv, iv, tv = g[nr], i[nr], tree_of[nr]
    par = bounded(draw4(seed, STREAM_TREE_PARENT, gv.astype(U64))[0], iv.astype(U64)).astype(np.int64)
    o = ebase[tv] + iv - 1
    pairs[o, 0] = gv
    pairs[o, 1] = base[tv] + par
    if extra:
        te = np.repeat(np.arange(trees, dtype=np.int64), extra)
        ee = np.tile(np.arange(extra, dtype=np.int64), trees)
        r0, r1, _, _ = draw4(seed, STREAM_TREE_EXTRA, (te * extra + ee).astype(U64))
        s = sizes[te].astype(U64)
        o = ebase[te] + sizes[te] - 1 + ee
        pairs[o, 0] = base[te] + bounded(r0, s).astype(np.int64)
        pairs[o, 1] = base[te] + bounded(r1, s).astype(np.int64)
    if permute:
        pairs = permutation(n, seed)[pairs]
    return n, pairs


def baseline_graph(index: int):
    """(n, pairs) of BASELINE.json configs[index-1], seed 0 (generators.baseline_graph)."""
    if index == 1:
        n, m = 1 << 16, 1 << 20
        return n, np.random.default_rng(0).integers(0, n, (m, 2)).astype(np.int32)
    if index == 2:
        return rmat(22, 16, seed=0)
    if index == 3:
        return grid(4096, 4096, 0.4, seed=0)
    if index == 4:
        return forest(1 << 20, 1, 64, 2, seed=0)
    raise ValueError(f"config {index}: the reference is infeasible at this size (SURVEY §8c)")


def csr(n: int, pairs: np.ndarray):
    """Symmetric, deduplicated, self-loop-free CSR with sorted rows
    (svcc.build_csr semantics, graph.py:55-97): int64 offsets and columns."""
    u = pairs[:, 0].astype(np.int64)
    v = pairs[:, 1].astype(np.int64)
    keep = u != v
    u, v = u[keep], v[keep]
    rows = np.concatenate([u, v])
    cols = np.concatenate([v, u])
    del u, v
    bits = max(1, int(n - 1).bit_length())
    keys = (rows << bits) | cols
    del rows, cols
    # bucket by the top row bits (stable radix argsort of a uint16), then sort
    # and dedupe each bucket on the thread pool
    nb_bits = min(12, bits)
    bucket = (keys >> (2 * bits - nb_bits)).astype(np.uint16)
    order = np.argsort(bucket, kind="stable")
    keys = keys[order]
    del order
    edges = np.concatenate([[0], np.cumsum(np.bincount(bucket, minlength=1 << nb_bits))])
    del bucket
    parts = [None] * (len(edges) - 1)

    def sort_bucket(k):
        seg = np.sort(keys[edges[k]:edges[k + 1]])
        if seg.size:
            seg = seg[np.concatenate([[True], seg[1:] != seg[:-1]])]
        parts[k] = seg

    with ThreadPoolExecutor(threads()) as ex:
        list(ex.map(sort_bucket, range(len(parts))))
    keys = np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)
    row = keys >> bits
    col = keys & ((1 << bits) - 1)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(row, minlength=n), out=off[1:])
    return off, col.astype(np.int64)
