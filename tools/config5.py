"""Config 5 (RMAT-27, edgefactor 16: 2^31 undirected edges, ~4.3e9 directed
entries, int64 offsets) on ONE B200: generation, host CSR build, upload,
solves, and a bit-exact check against the C oracle (the Python reference is
infeasible at this size). Prints one JSON line.

    python tools/config5.py [--scale 27] [--no-oracle]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=27)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import paper_1910_05971_b200 as fb
    from paper_1910_05971_b200 import generators as gen
    out = {"config": 5, "scale": a.scale, "host_cores": len(os.sched_getaffinity(0))}
    t = time.time()
    n, pairs = gen.rmat(a.scale, 16, seed=0)
    out["gen_s"] = round(time.time() - t, 1)
    out["n"], out["edges"] = n, int(pairs.shape[0])
    out["pairs_digest"] = gen.pairs_digest(pairs)
    t = time.time()
    g = fb.build_csr(n, pairs)
    out["csr_build_s"] = round(time.time() - t, 1)
    out["m_dir"] = g.m
    del pairs
    s = fb.Solver(0)
    t = time.time()
    s.upload(g)
    out["upload_s"] = round(time.time() - t, 2)
    times = []
    for _ in range(a.reps):
        st = s.solve()
        times.append(st.solve_ms)
    out["iterations"] = int(st.iterations)
    out["sparse_iterations"] = int(st.sparse_iterations)
    out["solve_ms"] = [round(x, 3) for x in times]
    best = min(times[1:]) if len(times) > 1 else times[0]
    out["edges_per_s"] = out["edges"] / (best * 1e-3)
    bi = 4 * g.m + 8 * (n + 1) + 24 * n
    out["iteration_model_frac"] = st.iterations * bi / (best * 1e-3) / 6553.3e9
    pr = s.solve(profile=True)
    out["profile_ms"] = {"first": pr.first_ms, "hook_dense": pr.hook_ms, "push": pr.push_ms,
                         "hubfix": pr.hubfix_ms, "shortcut": pr.shortcut_ms, "total": pr.solve_ms}
    labels = s.labels()
    gfc, fc, ms = s.trace()
    out["gf_changed"] = gfc.tolist()
    out["components"] = int(s.stats.component_count)
    out["labels_digest"] = gen.pairs_digest(labels)
    s.close()
    if not a.no_oracle:
        import oracle
        t = time.time()
        o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, cap=64)
        out["oracle_s"] = round(time.time() - t, 1)
        out["oracle_iterations"] = o.iterations
        out["parity"] = bool(o.iterations == out["iterations"] and np.array_equal(o.labels, labels)
                             and o.gf_changed.tolist() == out["gf_changed"])
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
