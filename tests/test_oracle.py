"""The CPU oracle (oracle/) pinned to the reference's own outputs.

Golden vectors come from the reference itself (tests/golden/make_golden.py):
379 graphs (the reference fixture families, random multigraphs with
self-loops/duplicates, small instances of the config generators) with
iteration counts, gf_changed/f_changed traces and every per-iteration parent
vector, plus BASELINE configs 1-4 at full size (traces + label digests)."""

import numpy as np
import pytest

import oracle
from oracle import port
from golden_io import load_configs, load_kats, load_suite
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen

SUITE = load_suite()


def test_suite_size():
    assert len(SUITE) >= 370
    names = {c.name for c in SUITE}
    assert {"path64", "star10", "complete64", "grid7x9", "mix50", "rmat12", "forest256"} <= names


@pytest.mark.parametrize("fn", [oracle.fastsv_csr, oracle.fastsv_la_csr])
def test_oracle_csr_matches_reference(fn):
    for c in SUITE:
        g = fb.build_csr(c.n, c.edges)
        assert g.m == c.m_dir, c.name
        r = fn(c.n, g.row_offsets, g.col_indices, snapshots=True)
        assert r.iterations == c.iterations, c.name
        assert r.gf_changed.tolist() == c.gf_changed, c.name
        assert r.f_changed.tolist() == c.f_changed, c.name
        assert np.array_equal(r.labels, c.labels), c.name
        assert np.array_equal(r.snapshots, c.snapshots), c.name


def test_oracle_raw_edges_matches_reference():
    # E3: self-loops and duplicates in the raw list change no snapshot
    for c in SUITE:
        r = oracle.fastsv_edges(c.n, c.edges, snapshots=True)
        assert r.iterations == c.iterations, c.name
        assert np.array_equal(r.snapshots, c.snapshots), c.name


def test_union_find_matches_reference():
    for c in SUITE:
        assert np.array_equal(oracle.uf_labels(c.n, c.edges), c.labels), c.name


@pytest.mark.parametrize("mode,threshold,workers", [("auto", 0.1, 1), ("auto", 1.0, 3),
                                                    ("dense_only", 0.1, 2), ("sparse_only", 0.1, 1),
                                                    ("auto", 0.0, 1)])
def test_numpy_port_matches_reference(mode, threshold, workers):
    for c in SUITE[::3]:
        g = fb.build_csr(c.n, c.edges)
        f, it, gfc, kinds = port.fastsv_la(port.PortGraph(c.n, g.row_offsets, g.col_indices),
                                           threshold=threshold, workers=workers, mode=mode)
        assert it == c.iterations and gfc == c.gf_changed, c.name
        assert np.array_equal(f, c.labels), c.name
        assert kinds[0] == ("sparse" if mode == "sparse_only" else "dense")


def test_reference_kats():
    k = load_kats()
    assert k["two_triangles"]["labels"] == [0, 0, 0, 3, 3, 3]
    g = fb.build_csr(10, [(0, i) for i in range(1, 10)])
    r = oracle.fastsv_csr(10, g.row_offsets, g.col_indices)
    assert r.iterations == k["star10"]["iterations"] == 2
    g = fb.build_csr(64, [(i, i + 1) for i in range(63)])
    assert oracle.fastsv_csr(64, g.row_offsets, g.col_indices).iterations == k["path64_fastsv"]["iterations"]


@pytest.mark.parametrize("index", [1, 2, 3, 4])
def test_baseline_configs_match_reference(index):
    rec = load_configs().get(index)
    if rec is None:
        pytest.skip(f"config {index} golden not generated (make_golden.py --full)")
    n, pairs = gen.baseline_graph(index)
    assert n == rec["n"] and pairs.shape[0] == rec["edges"]
    assert gen.pairs_digest(pairs) == rec["pairs_digest"]
    g = fb.build_csr(n, pairs)
    assert g.m == rec["m_dir"]
    r = oracle.fastsv_csr(n, g.row_offsets, g.col_indices)
    assert r.iterations == rec["iterations"]
    assert r.gf_changed.tolist() == rec["gf_changed"]
    assert r.f_changed.tolist() == rec["f_changed"]
    assert gen.pairs_digest(r.labels) == rec["labels_digest"]
    assert len(np.unique(r.labels)) == rec["component_count"]
