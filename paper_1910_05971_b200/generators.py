"""Synthetic inputs of BASELINE.json's five configs (the reference has no
generator for any of them). Streams are pinned: configs 2-5 by
the counter-based Philox generators of include/fsv_graphgen.h, config 1 by
numpy's PCG64 ``default_rng(0).integers(0, n, (m, 2))`` (the survey probe's
definition, BASELINE.json configs[0]).

Every generator returns ``(n, pairs)`` with ``pairs`` an int32 array of shape
(m, 2) — self-loops and duplicates kept, as raw edge lists are.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._native import graphgen_lib

RMAT_ABC = (0.57, 0.19, 0.19)


def set_threads(threads: int) -> None:
    graphgen_lib().fsvg_set_threads(int(threads))


def gnm_uniform(n: int, m: int, seed: int = 0):
    """G(n, m) with i.i.d. uniform endpoints (config 1)."""
    rng = np.random.default_rng(seed)
    return n, rng.integers(0, n, (m, 2)).astype(np.int32)


def rmat(scale: int, edgefactor: int = 16, abc=RMAT_ABC, seed: int = 0, permute: bool = True):
    """RMAT, one 32-bit Philox draw per level per edge, ids permuted."""
    n = 1 << scale
    m = edgefactor * n
    pairs = np.empty((m, 2), dtype=np.int32)
    r = graphgen_lib().fsvg_rmat(scale, m, abc[0], abc[1], abc[2], seed, int(permute), pairs.ctypes.data)
    if r != m:
        raise ValueError(f"fsvg_rmat failed ({r})")
    return n, pairs


def grid(rows: int, cols: int, p_drop: float = 0.4, seed: int = 0, permute: bool = True):
    """rows x cols 4-neighbour grid, each edge dropped with probability p."""
    L = graphgen_lib()
    m = L.fsvg_grid(rows, cols, p_drop, seed, int(permute), None)
    if m < 0:
        raise ValueError("fsvg_grid failed")
    pairs = np.empty((m, 2), dtype=np.int32)
    r = L.fsvg_grid(rows, cols, p_drop, seed, int(permute), pairs.ctypes.data)
    if r != m:
        raise ValueError("fsvg_grid failed")
    return rows * cols, pairs


def forest(trees: int, min_size: int = 1, max_size: int = 64, extra: int = 2, seed: int = 0,
           permute: bool = True):
    """Random recursive trees with sizes U[min, max] plus `extra` intra-tree pairs."""
    L = graphgen_lib()
    n = ctypes.c_int64(0)
    m = L.fsvg_forest(trees, min_size, max_size, extra, seed, int(permute), None, ctypes.byref(n))
    if m < 0:
        raise ValueError("fsvg_forest failed")
    pairs = np.empty((m, 2), dtype=np.int32)
    r = L.fsvg_forest(trees, min_size, max_size, extra, seed, int(permute), pairs.ctypes.data,
                      ctypes.byref(n))
    if r != m:
        raise ValueError("fsvg_forest failed")
    return int(n.value), pairs


def pairs_digest(pairs: np.ndarray) -> str:
    a = np.ascontiguousarray(pairs, dtype=np.int32)
    return f"{graphgen_lib().fsvg_fnv1a64(a.ctypes.data, a.nbytes):016x}"


@dataclass(frozen=True)
class BaselineConfig:
    index: int
    name: str
    description: str

    def generate(self, scale_override: int | None = None):
        return baseline_graph(self.index, scale_override)


CONFIGS = {
    1: BaselineConfig(1, "gnm-2^16-2^20", "G(n=2^16, m=2^20) uniform endpoints, seed 0"),
    2: BaselineConfig(2, "rmat22-ef16", "RMAT scale 22, edgefactor 16, .57/.19/.19/.05, permuted"),
    3: BaselineConfig(3, "grid4096-p0.4", "4096x4096 grid, edges dropped w.p. 0.4, permuted"),
    4: BaselineConfig(4, "forest-2^20", "2^20 random trees, sizes U[1,64], +2 edges/tree, permuted"),
    5: BaselineConfig(5, "rmat27-ef16", "RMAT scale 27, edgefactor 16, .57/.19/.19/.05, permuted"),
}


def baseline_graph(index: int, scale_override: int | None = None):
    """(n, pairs) of BASELINE.json configs[index-1], seed 0."""
    if index == 1:
        return gnm_uniform(1 << 16, 1 << 20, seed=0)
    if index == 2:
        return rmat(scale_override or 22, 16, seed=0)
    if index == 3:
        side = 4096 if scale_override is None else 1 << (scale_override // 2)
        return grid(side, side, 0.4, seed=0)
    if index == 4:
        return forest(1 << (scale_override or 20), 1, 64, 2, seed=0)
    if index == 5:
        return rmat(scale_override or 27, 16, seed=0)
    raise ValueError(f"unknown config {index}")
