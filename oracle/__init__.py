"""CPU parity oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline — never as the thing shipped. The product path
(``paper_1910_05971_b200``) never imports it and has no CPU fallback.

Contents
  fsv_oracle.c   plain-C restatement of the reference algorithms
                 (union-find oracle.py:12-55; FastSV algorithms.py:79-142;
                 fastsv_la driver.py:64-120) — wrapped below.
  port.py        numpy restatement of the reference's own CPU hot path
                 (kernels.py + driver.py), used as the timed CPU baseline.

Parity of both against the reference itself is pinned by tests/test_oracle.py
through golden vectors the reference produced (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "liboracle.so"
_lib = None

ORC_ERR_INVARIANT = 3


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            import sys
            sys.path.insert(0, str(_HERE.parent))
            from paper_1910_05971_b200.build import build_oracle
            build_oracle()
        L = ctypes.CDLL(str(LIB_PATH))
        P, I = ctypes.c_void_p, ctypes.c_int64
        L.oracle_uf_labels.argtypes = [I, I, P, P]
        for name in ("oracle_fastsv_csr", "oracle_fastsv_la_csr"):
            getattr(L, name).argtypes = [I, P, P, I, P, P, P, P, P]
        L.oracle_fastsv_edges.argtypes = [I, I, P, I, P, P, P, P, P]
        _lib = L
    return _lib


class OracleResult:
    def __init__(self, labels, iterations, gf_changed, f_changed, snapshots):
        self.labels = labels
        self.iterations = iterations
        self.gf_changed = gf_changed
        self.f_changed = f_changed
        self.snapshots = snapshots


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else None


def uf_labels(n: int, pairs) -> np.ndarray:
    """Union-find + min relabel (oracle.py:39-55): int32 labels."""
    pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
    out = np.empty(n, dtype=np.int32)
    rc = lib().oracle_uf_labels(n, pairs.shape[0], _ptr(pairs), _ptr(out))
    if rc:
        raise ValueError(f"oracle_uf_labels failed ({rc})")
    return out


def _run(fn, n, args, cap, snapshots):
    labels = np.empty(n, dtype=np.int32)
    it = np.zeros(1, dtype=np.int64)
    gfc = np.zeros(cap, dtype=np.int64)
    fc = np.zeros(cap, dtype=np.int64)
    snaps = np.empty((cap, n), dtype=np.int32) if snapshots else None
    rc = fn(n, *args, cap, _ptr(labels), _ptr(it), _ptr(gfc), _ptr(fc), _ptr(snaps) if snapshots else None)
    if rc == ORC_ERR_INVARIANT:
        raise AssertionError("oracle invariant violated")
    if rc:
        raise ValueError(f"oracle failed ({rc})")
    k = int(it[0])
    return OracleResult(labels, k, gfc[:min(k, cap)], fc[:min(k, cap)],
                        snaps[:min(k, cap)] if snapshots else None)


def fastsv_csr(n, offsets, cols, cap=4096, snapshots=False) -> OracleResult:
    """All-flags FastSV, edge-parallel form (algorithms.py:79-91, 117-142)."""
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    return _run(lib().oracle_fastsv_csr, n, (_ptr(offsets), _ptr(cols)), cap, snapshots)


def fastsv_la_csr(n, offsets, cols, cap=4096, snapshots=False) -> OracleResult:
    """Matrix formulation (driver.py:64-120) with dense products."""
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    return _run(lib().oracle_fastsv_la_csr, n, (_ptr(offsets), _ptr(cols)), cap, snapshots)


def fastsv_edges(n, pairs, cap=4096, snapshots=False) -> OracleResult:
    """FastSV over a raw pair list (self-loops / duplicates kept, E3)."""
    pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
    return _run(lib().oracle_fastsv_edges, n, (pairs.shape[0], _ptr(pairs)), cap, snapshots)
