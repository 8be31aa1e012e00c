"""GPU parity: the sm_100a path through the C ABI against the CPU oracle
(itself pinned to the reference's golden vectors in test_oracle.py).

Bar: bit-exact labels, iteration count, gf_changed and f_changed traces and
every per-iteration parent vector (snapshot)."""

import numpy as np
import pytest

import oracle
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
from conftest import random_multigraph

pytestmark = pytest.mark.gpu


def check_against_oracle(solver, n, pairs, snapshots=True, hub_slots=0):
    g = fb.build_csr(n, pairs)
    solver.set_hub_slots(hub_slots)
    solver.upload(g)
    labels, iters, gfc, fc, ms, snaps = solver.run(snapshots=snapshots, snap_cap=512)
    o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, snapshots=snapshots)
    assert iters == o.iterations
    assert gfc.tolist() == o.gf_changed.tolist()
    assert fc.tolist() == o.f_changed.tolist()
    assert np.array_equal(labels, o.labels)
    if snapshots:
        for k in range(iters):
            assert np.array_equal(snaps[k], o.snapshots[k]), f"snapshot {k + 1} differs"
    return g, labels, iters


def test_random_multigraphs_snapshots(solver):
    rng = np.random.default_rng(71)
    for _ in range(200):
        n, pairs = random_multigraph(rng, max_n=40, density=2.5)
        check_against_oracle(solver, n, pairs)


def test_random_with_forced_hubs(solver):
    # hub table forced on small graphs: every column-side path (hub / non-hub)
    rng = np.random.default_rng(72)
    for _ in range(100):
        n = int(rng.integers(300, 3000))
        k = int(rng.integers(n, 20 * n))
        # skewed endpoints so some vertices pass the hub degree threshold
        u = (rng.pareto(1.2, k) * 3).astype(np.int64) % n
        v = rng.integers(0, n, k)
        pairs = np.stack([u, v], 1).astype(np.int32)
        check_against_oracle(solver, n, pairs, snapshots=True, hub_slots=0)


def test_edge_cases(solver):
    for n, pairs in [(1, []), (2, []), (5, [(0, 0), (1, 1)]), (2, [(0, 1)]), (3, [(2, 1)]),
                     (6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)]),
                     (64, [(i, i + 1) for i in range(63)]),
                     (10, [(0, i) for i in range(1, 10)])]:
        p = np.asarray(pairs, dtype=np.int32).reshape(-1, 2)
        check_against_oracle(solver, n, p)


def test_two_triangles_labels():
    r = fb.fastsv_la(fb.build_csr(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)]))
    assert r.labeling.labels.tolist() == [0, 0, 0, 3, 3, 3]


def test_star10_two_iterations():
    r = fb.fastsv(fb.build_csr(10, [(0, i) for i in range(1, 10)]))
    assert r.iterations == 2
    assert r.labeling.labels.tolist() == [0] * 10


@pytest.mark.parametrize("scale", [12, 16])
def test_rmat_small(solver, scale):
    n, pairs = gen.rmat(scale, 16, seed=3)
    check_against_oracle(solver, n, pairs, snapshots=True)


def test_config1_full(solver):
    n, pairs = gen.baseline_graph(1)
    g, labels, iters = check_against_oracle(solver, n, pairs, snapshots=False)
    assert np.array_equal(labels, oracle.uf_labels(n, pairs))
