"""Generate the golden vectors that pin the oracle (and through it the GPU
path) to the REFERENCE implementation itself.

Run here, where the reference is importable (it is not on the GPU box):

    python tests/golden/make_golden.py            # small suite + config 1 + small families
    python tests/golden/make_golden.py --full     # also configs 2-4 at BASELINE size

Every value below is produced by /root/reference/pkg/src/svcc (read-only,
imported unchanged): ``svcc.fastsv_la(..., record_snapshots=True)`` for
iteration counts, gf_changed/f_changed traces and per-iteration parent
vectors; ``svcc.union_find_labels`` for labels; ``svcc.build_csr`` for the
CSR layout. The graphs are the reference's own fixture families
(pkg/tests/conftest.py:19-38 via svcc.generate), random multigraphs shaped
like pkg/tests/conftest.py:62-72, and small instances of this repo's
generators for configs 2-4 (whose streams are pinned by digests here).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import svcc  # noqa: E402  (the reference)

from paper_1910_05971_b200 import build_csr  # noqa: E402
from paper_1910_05971_b200 import generators as gen  # noqa: E402


def reference_run(n, edges):
    """All reference outputs for one raw edge list."""
    g = svcc.build_csr(n, edges)
    r = svcc.fastsv_la(g, record_snapshots=True)
    uf = svcc.union_find_labels(n, np.asarray(edges).reshape(-1, 2)).labels
    assert np.array_equal(uf, r.labeling.labels)
    return g, r


def suite_cases():
    """(name, n, int32 edges) — the reference fixture families plus random
    multigraphs with self-loops and duplicates."""
    cases = []
    specs = []
    for n in range(1, 65):
        specs += [(f"path{n}", svcc.GeneratorSpec("path", n=n)),
                  (f"cycle{n}", svcc.GeneratorSpec("cycle", n=n)),
                  (f"star{n}", svcc.GeneratorSpec("star", n=n))]
    for n in (2, 3, 4, 5, 8, 13, 21, 34, 55, 64):
        specs.append((f"complete{n}", svcc.GeneratorSpec("complete", n=n)))
    for r, c in ((2, 2), (3, 3), (4, 4), (5, 5), (8, 8), (2, 32), (4, 16), (7, 9)):
        specs.append((f"grid{r}x{c}", svcc.GeneratorSpec("grid2d", rows=r, cols=c)))
    sizes = (200, 500, 1000, 2000)
    for p in (0.002, 0.01, 0.05):
        for seed in range(20):
            n = sizes[seed % 4]
            if n <= 500:
                specs.append((f"gnp-n{n}-p{p}-s{seed}", svcc.GeneratorSpec("gnp", n=n, p=p, seed=seed)))
    for blocks in range(2, 51, 4):
        specs.append((f"mix{blocks}", svcc.GeneratorSpec("component_mix", blocks=blocks, block_n=30,
                                                         block_p=0.1, seed=1000 + blocks)))
    for name, spec in specs:
        g = svcc.generate(spec)
        keep = g.row_ids < g.col_indices
        e = np.stack([g.row_ids[keep], g.col_indices[keep]], 1).astype(np.int32)
        cases.append((name, g.n, e))
    rng = np.random.default_rng(20261020)
    for i in range(120):
        n = int(rng.integers(1, 41))
        k = int(rng.integers(0, int(2.5 * n) + 1))
        cases.append((f"multi{i}", n, rng.integers(0, n, (k, 2)).astype(np.int32)))
    # small instances of the BASELINE config families (this repo's generators)
    for scale in (8, 10, 12):
        n, e = gen.rmat(scale, 16, seed=5)
        cases.append((f"rmat{scale}", n, e))
    n, e = gen.grid(48, 48, 0.4, seed=5)
    cases.append(("grid48-p0.4", n, e))
    n, e = gen.grid(96, 64, 0.4, seed=6)
    cases.append(("grid96x64-p0.4", n, e))
    n, e = gen.forest(256, 1, 64, 2, seed=5)
    cases.append(("forest256", n, e))
    return cases


def make_suite():
    names, ns, e_off, i_off, s_off = [], [], [0], [0], [0]
    edges, iters, gfc, fc, labels, snaps, mdir = [], [], [], [], [], [], []
    for name, n, e in suite_cases():
        g, r = reference_run(n, e)
        names.append(name)
        ns.append(n)
        edges.append(e.reshape(-1))
        e_off.append(e_off[-1] + e.size)
        iters.append(r.iterations)
        gfc += [t.gf_changed for t in r.trace]
        fc += [t.f_changed for t in r.trace]
        i_off.append(i_off[-1] + r.iterations)
        labels.append(r.labeling.labels.astype(np.int32))
        snaps.append(np.concatenate([s.astype(np.int32) for s in r.snapshots]) if n else
                     np.zeros(0, np.int32))
        s_off.append(s_off[-1] + n * r.iterations)
        mdir.append(g.m)
    np.savez_compressed(
        HERE / "suite.npz",
        names=np.array(names), n=np.array(ns, np.int64), m_dir=np.array(mdir, np.int64),
        edges=np.concatenate(edges).astype(np.int32), edge_off=np.array(e_off, np.int64),
        iterations=np.array(iters, np.int64), gf_changed=np.array(gfc, np.int64),
        f_changed=np.array(fc, np.int64), trace_off=np.array(i_off, np.int64),
        labels=np.concatenate(labels).astype(np.int32),
        snapshots=np.concatenate(snaps).astype(np.int32), snap_off=np.array(s_off, np.int64))
    print(f"suite: {len(names)} graphs")


DRIVER_CONFIGS = {
    "auto": dict(),
    "auto_t1": dict(sparse_threshold=1.0),
    "auto_t05": dict(sparse_threshold=0.5),
    "sparse_only": dict(force_kernel="sparse_only"),
    "dense_only": dict(force_kernel="dense_only"),
}


def make_driver_traces():
    """Reference IterationTrace.kernel / .flops under several DriverConfigs
    (driver.py:51-61, 85-93; kernels.py:67-68, 94-102) for a subset of the
    suite: the device reproduces the same product schedule."""
    cases = suite_cases()[::4]
    names, kinds, flops, off = [], [], [], [0]
    for cname, cfg in DRIVER_CONFIGS.items():
        for name, n, e in cases:
            g = svcc.build_csr(n, e)
            r = svcc.fastsv_la(g, svcc.DriverConfig(**cfg))
            names.append(f"{cname}:{name}")
            kinds += [1 if t.kernel == "sparse" else 0 for t in r.trace]
            flops += [t.flops for t in r.trace]
            off.append(off[-1] + r.iterations)
    np.savez_compressed(HERE / "driver_traces.npz", names=np.array(names),
                        kernel=np.array(kinds, np.int32), flops=np.array(flops, np.int64),
                        off=np.array(off, np.int64))
    print(f"driver traces: {len(names)} runs")


def kats():
    """Known-answer tests quoted from the reference's own tests."""
    out = {}
    r = svcc.fastsv_la(svcc.build_csr(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)]))
    out["two_triangles"] = {"labels": r.labeling.labels.tolist()}            # test_driver.py:52-57
    r = svcc.fastsv(svcc.build_csr(10, [(0, i) for i in range(1, 10)]))
    out["star10"] = {"iterations": r.iterations, "labels": r.labeling.labels.tolist()}  # test_algorithms.py:97-103
    r = svcc.fastsv(svcc.generate(svcc.GeneratorSpec("path", n=64)))
    out["path64_fastsv"] = {"iterations": r.iterations}
    (HERE / "kats.json").write_text(json.dumps(out, indent=1))
    print("kats:", out["star10"]["iterations"], out["path64_fastsv"]["iterations"])


def config_record(index, full_labels=False):
    """Reference outputs at BASELINE size for config `index` (CSR from the
    repo's builder, checked equal to svcc.build_csr on config 1)."""
    t0 = time.time()
    n, pairs = gen.baseline_graph(index)
    g = build_csr(n, pairs)
    if index == 1:
        gref = svcc.build_csr(n, pairs.astype(np.int64))
        assert np.array_equal(gref.row_offsets, g.row_offsets)
        assert np.array_equal(gref.col_indices, g.col_indices)
    rg = svcc.CsrGraph(n=n, row_offsets=g.row_offsets.astype(np.int64),
                       col_indices=g.col_indices.astype(np.int64))
    r = svcc.fastsv_la(rg)
    labels = r.labeling.labels.astype(np.int32)
    rec = {
        "config": index, "n": n, "edges": int(pairs.shape[0]), "m_dir": g.m,
        "pairs_digest": gen.pairs_digest(pairs),
        "iterations": r.iterations,
        "gf_changed": [t.gf_changed for t in r.trace],
        "f_changed": [t.f_changed for t in r.trace],
        "component_count": r.labeling.component_count,
        "labels_digest": gen.pairs_digest(labels),
        "reference_fastsv_la_seconds": round(time.time() - t0, 1),
    }
    if index == 1:
        uf = svcc.union_find_labels(n, pairs.astype(np.int64)).labels
        assert np.array_equal(uf, r.labeling.labels)
        rec["union_find_checked"] = True
    print(json.dumps(rec))
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true", help="also configs 2-4 at full size (minutes)")
    args = ap.parse_args()
    make_suite()
    make_driver_traces()
    kats()
    recs = {1: config_record(1)}
    path = HERE / "configs.json"
    if path.exists():
        old = json.loads(path.read_text())
        for k, v in old.items():
            recs.setdefault(int(k), v)
    if args.full:
        for i in (2, 3, 4):
            recs[i] = config_record(i)
    path.write_text(json.dumps({str(k): v for k, v in sorted(recs.items())}, indent=1))


if __name__ == "__main__":
    main()
