"""Graph and label containers of the drop-in (mirrors svcc.graph,
/root/reference/pkg/src/svcc/graph.py).

``CsrGraph`` keeps the reference's invariants (symmetric, deduplicated,
self-loop free, rows sorted; graph.py:24-27). Row offsets are int64 like the
reference; column ids are int32 here (the device id type) — ``fastsv_la``
also accepts a reference ``svcc.CsrGraph`` with int64 columns unchanged.
``build_csr`` runs the OpenMP host builder of include/fsv_graphgen.h.
"""

from __future__ import annotations

from collections.abc import Mapping
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np

from ._native import graphgen_lib
from .errors import InputError, InvariantError

ID_DTYPE = np.int64      # labels / offsets, as the reference (graph.py:15-17)
COL_DTYPE = np.int32     # device column id type


@dataclass(frozen=True)
class CsrGraph:
    """Symmetric adjacency in CSR form (graph.py:20-52)."""

    n: int
    row_offsets: np.ndarray
    col_indices: np.ndarray

    @property
    def m(self) -> int:
        """Stored directed entries; an undirected edge contributes two."""
        return int(self.col_indices.size)

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    def neighbors(self, u: int) -> np.ndarray:
        lo, hi = self.row_offsets[u], self.row_offsets[u + 1]
        return self.col_indices[lo:hi]

    @cached_property
    def row_ids(self) -> np.ndarray:
        out = np.repeat(np.arange(self.n, dtype=ID_DTYPE), self.degrees)
        out.flags.writeable = False
        return out


def _as_pairs(edges) -> np.ndarray:
    if isinstance(edges, np.ndarray):
        pairs = edges
    else:
        pairs = np.asarray(list(edges), dtype=ID_DTYPE)
    if pairs.size == 0:
        pairs = pairs.reshape(0, 2)
    if pairs.ndim != 2 or pairs.shape[1] != 2:
        raise InputError("edges must be (u, v) pairs")
    return pairs


def build_csr(n, edges) -> CsrGraph:
    """Symmetric deduplicated CSR from an edge list (graph.py:55-97 semantics:
    range check -> drop self-loops -> both orientations -> unique -> sorted
    rows). Accepts an iterable of pairs or an integer array of shape (k, 2)."""
    if n < 0:
        raise InputError(f"vertex count must be non-negative, got {n}")
    if n > np.iinfo(np.int32).max:
        raise InputError(f"vertex count {n} exceeds the int32 id range")
    pairs = _as_pairs(edges)
    if pairs.dtype == np.int32:
        fn = graphgen_lib().fsvg_csr_build
    else:
        if pairs.dtype.kind not in "iu":
            pairs = pairs.astype(ID_DTYPE)
        pairs = pairs.astype(np.int64, copy=False)
        fn = graphgen_lib().fsvg_csr_build64
    pairs = np.ascontiguousarray(pairs)
    k = pairs.shape[0]
    offsets = np.empty(int(n) + 1, dtype=ID_DTYPE)
    cols = np.empty(max(2 * k, 1), dtype=COL_DTYPE)
    import ctypes
    bad = ctypes.c_int64(-1)
    m_dir = fn(int(n), k, pairs.ctypes.data, offsets.ctypes.data, cols.ctypes.data, ctypes.byref(bad))
    if m_dir < 0:
        if bad.value >= 0:
            u, v = pairs[bad.value]
            raise InputError(f"edge ({u}, {v}) out of range for n={n}")
        raise InputError("CSR build failed")
    cols = np.ascontiguousarray(cols[:m_dir]) if m_dir < cols.size else cols[:m_dir]
    offsets.flags.writeable = False
    cols.flags.writeable = False
    return CsrGraph(n=int(n), row_offsets=offsets, col_indices=cols)


class ComponentSizes(Mapping):
    """``Labeling.sizes`` (representative -> vertex count) backed by the arrays
    the device computed (fsv_get_labeling): representatives ascending, sizes
    aligned. Behaves as the reference's read-only dict (lookup, iteration in
    ascending representative order, len, equality with a dict); a dict is
    only built when one is iterated as items."""

    __slots__ = ("_reps", "_counts")

    def __init__(self, reps: np.ndarray, counts: np.ndarray):
        self._reps = reps
        self._counts = counts

    @property
    def representatives(self) -> np.ndarray:
        return self._reps

    @property
    def counts(self) -> np.ndarray:
        return self._counts

    def __getitem__(self, key):
        i = int(np.searchsorted(self._reps, key))
        if i < self._reps.size and self._reps[i] == key:
            return int(self._counts[i])
        raise KeyError(key)

    def __len__(self):
        return int(self._reps.size)

    def __iter__(self):
        return iter(self._reps.tolist())

    def items(self):
        return zip(self._reps.tolist(), self._counts.tolist())

    def __eq__(self, other):
        if isinstance(other, ComponentSizes):
            return np.array_equal(self._reps, other._reps) and np.array_equal(self._counts, other._counts)
        if isinstance(other, Mapping):
            return len(self) == len(other) and dict(self.items()) == dict(other.items())
        return NotImplemented

    __hash__ = None

    def __repr__(self):
        return f"ComponentSizes({len(self)} components)"


@dataclass(frozen=True)
class Labeling:
    """Final component labels: representative = minimum id (graph.py:100-106)."""

    labels: np.ndarray
    component_count: int
    sizes: dict = field(compare=False)


def labeling_from_parents(f: np.ndarray) -> Labeling:
    """Finalize a converged parent vector (graph.py:109-125)."""
    f = np.asarray(f, dtype=ID_DTYPE)
    if f.size and not np.array_equal(f[f], f):
        raise InvariantError("algorithm terminated on non-star forest")
    reps, counts = np.unique(f, return_counts=True)
    labels = f.copy()
    labels.flags.writeable = False
    return Labeling(labels=labels, component_count=int(reps.size),
                    sizes={int(r): int(c) for r, c in zip(reps, counts)})
