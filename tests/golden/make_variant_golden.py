"""Golden traces of the REFERENCE's weaker hooking variants (the sv1..sv5
ablation, algorithms.py:28-35,66-114,145-199) for the device variant path.
Run here, where the reference is importable (it is not on the GPU box):

    python tests/golden/make_variant_golden.py

For every golden-suite graph (plus four larger generated graphs) and every HookingConfig (16 flag combinations,
code = grandparent | stochastic << 1 | aggressive << 2 | early_termination << 3)
plus simplified_sv (code 16), svcc.fastsv / svcc.simplified_sv with
record_snapshots=True gives: iteration count, gf_changed and f_changed per
iteration, and a digest of the snapshots (every committed f as int64 bytes).
Writes tests/golden/variants.npz.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

import svcc  # noqa: E402  (the reference)
from svcc.algorithms import HookingConfig, simplified_sv  # noqa: E402

from golden_io import load_suite  # noqa: E402
from paper_1910_05971_b200 import generators as gen  # noqa: E402

SIMPLIFIED = 16


def extra_graphs():
    """Larger graphs from this repo's seeded generators (regenerated on the
    GPU side; their pair streams are pinned by digest)."""
    return [("x:config1", *gen.baseline_graph(1)), ("x:rmat14", *gen.rmat(14, 16, seed=5)),
            ("x:grid300", *gen.grid(300, 300, 0.4, seed=3)), ("x:forest2000", *gen.forest(2000, 1, 64, 2, seed=4))]


def flags(code):
    return HookingConfig(grandparent_hooking=bool(code & 1), stochastic_hooking=bool(code & 2),
                         aggressive_hooking=bool(code & 4), early_termination=bool(code & 8))


def snap_digest(snapshots):
    h = hashlib.sha256()
    for s in snapshots:
        h.update(np.ascontiguousarray(s, dtype="<i8").tobytes())
    return h.hexdigest()[:16]


def main():
    names, codes, iters, t_off, gfc, fc, digests = [], [], [], [0], [], [], []
    graphs = [(c.name, c.n, c.edges) for c in load_suite()] + extra_graphs()
    extra = {name: gen.pairs_digest(e) for name, _, e in extra_graphs()}
    for name, n, edges in graphs:
        g = svcc.build_csr(n, edges)
        for code in range(17):
            r = simplified_sv(g, True) if code == SIMPLIFIED else svcc.fastsv(g, flags(code), True)
            names.append(name)
            codes.append(code)
            iters.append(r.iterations)
            gfc.extend(t.gf_changed for t in r.trace)
            fc.extend(t.f_changed for t in r.trace)
            t_off.append(len(gfc))
            digests.append(snap_digest(r.snapshots))
    np.savez_compressed(HERE / "variants.npz", names=np.array(names), codes=np.array(codes, np.int32),
                        iterations=np.array(iters, np.int32), trace_off=np.array(t_off, np.int64),
                        gf_changed=np.array(gfc, np.int64), f_changed=np.array(fc, np.int64),
                        digests=np.array(digests), extra_names=np.array(list(extra)),
                        extra_digests=np.array(list(extra.values())))
    print(f"{len(names)} runs")


if __name__ == "__main__":
    main()
