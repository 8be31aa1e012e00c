"""numpy restatement of the device schedule of the hooking variants
(csrc/fsv_variants.cuh) — test-only. Same init forms and filters as the
kernels, so a CPU test can pin them to the reference's own variant traces
(tests/golden/variants.npz) before the GPU runs them."""

import hashlib

import numpy as np


def run(n, offsets, cols, code):
    """code: grandparent | stochastic << 1 | aggressive << 2 | early_term << 3,
    or 16 = simplified_sv. Returns (iterations, gf_changed, f_changed, snapshot digest)."""
    gp, sto, agg = bool(code & 1), bool(code & 2), bool(code & 4)
    if code == 16:
        gp = sto = agg = False
    gf_stop = code == 15
    offsets = np.asarray(offsets, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(offsets))
    cols = np.asarray(cols, dtype=np.int64)
    F = np.arange(n, dtype=np.int64)
    G = F.copy()
    h = hashlib.sha256()
    gfc, fc, it = [], [], 0
    while True:
        it += 1
        val = (G if gp else F)[cols]
        fu, gu = F[rows], G[rows]
        N = np.minimum(F, G) if sto else F.copy()
        sel = (sto | (gu == fu)) & (val < gu)              # N[f[u]] <-min val
        np.minimum.at(N, fu[sel], val[sel])
        if agg:
            sel = val < fu                                  # N[u] <-min val
            np.minimum.at(N, rows[sel], val[sel])
        P = N if sto else np.minimum(N, N[N])              # two-commit shortcut
        Gn = P[P]
        gfc.append(int(np.count_nonzero(Gn != G)))
        fc.append(int(np.count_nonzero(P != F)))
        assert not np.any(P > F)
        h.update(np.ascontiguousarray(P, dtype="<i8").tobytes())
        F, G = P, Gn
        if (gfc[-1] if gf_stop else fc[-1]) == 0:
            break
    return it, gfc, fc, h.hexdigest()[:16]
