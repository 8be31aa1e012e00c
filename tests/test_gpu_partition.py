"""The multi-GPU schedule's rank-partitioned CUDA kernels, run as an emulated
rank group on ONE device (fsv_group_solve): R contexts each hold one
contiguous row range of the graph (bench.row_partition, the 1D partition of
SURVEY §8e), every rank's hooking kernels run, one device kernel min-merges
the ranks' next-parent vectors in place of ncclAllReduce(min), then every
rank's vertex pass. No kernel waits on another (they run in order on one
stream), so this is safe with fewer GPUs than ranks.

This covers what the multi-process NCCL path runs per rank: the partitioned
oriented layout (global-degree orientation, each undirected edge kept by one
rank), per-rank hub tables and hub fix-up, the row-filtered sparse push, the
f_1 assembly by min-merge, and the host-batched loop. Bar: every
per-iteration parent vector, the trace and the labels equal the oracle's
(and the reference's golden vectors), and all ranks hold the same labels.
"""

import numpy as np
import pytest

import bench
import oracle
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
from paper_1910_05971_b200.driver import group_run
from golden_io import load_configs, load_suite

pytestmark = pytest.mark.gpu


def make_group(g, ranks, hub_slots=0):
    solvers = []
    for r in range(ranks):
        lo, hi = bench.row_partition(g.row_offsets, ranks, r)
        s = fb.Solver(0, hub_slots=hub_slots)
        s.upload(g, lo, hi, g.col_indices[g.row_offsets[lo]:g.row_offsets[hi]])
        solvers.append(s)
    return solvers


def close_all(solvers):
    for s in solvers:
        s.close()


def run_group(g, ranks, hub_slots=0, snapshots=True, policy=0, threshold=0.1, batch=0):
    solvers = make_group(g, ranks, hub_slots)
    try:
        out = group_run(solvers, snapshots=snapshots, snap_cap=512, policy=policy, threshold=threshold,
                        batch=batch)
    finally:
        close_all(solvers)
    return out


def check_oracle(n, g, ranks, hub_slots=0, policy=0, threshold=0.1, o=None):
    labels, iters, gfc, fc, snaps, kern, flops, all_labels = run_group(g, ranks, hub_slots, True, policy, threshold)
    if o is None:
        o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, snapshots=True)
    assert iters == o.iterations, (ranks, hub_slots, policy)
    assert gfc.tolist() == o.gf_changed.tolist() and fc.tolist() == o.f_changed.tolist()
    assert np.array_equal(labels, o.labels)
    for k in range(iters):
        assert np.array_equal(snaps[k], o.snapshots[k]), f"snapshot {k + 1} differs (R={ranks})"
    for lab in all_labels[1:]:
        assert np.array_equal(lab, labels), "ranks disagree"
    return kern, flops


@pytest.mark.parametrize("ranks", [2, 4])
def test_group_golden_suite_snapshots(ranks):
    """All 379 reference golden graphs, every per-iteration parent vector."""
    for c in load_suite():
        g = fb.build_csr(c.n, c.edges)
        labels, iters, gfc, fc, snaps, kern, flops, all_labels = run_group(g, ranks)
        assert iters == c.iterations, c.name
        assert gfc.tolist() == c.gf_changed and fc.tolist() == c.f_changed, c.name
        assert np.array_equal(labels, c.labels), c.name
        assert np.array_equal(snaps, c.snapshots), c.name
        assert all(np.array_equal(x, labels) for x in all_labels), c.name


@pytest.mark.parametrize("ranks", [2, 3, 4, 8])
def test_group_rmat_all_schedules(ranks):
    """RMAT-14 with the hub table: dense pulls, sparse pushes (row-filtered
    per rank) and the reference's auto schedule; trace flops summed over
    ranks equal the single-context trace."""
    n, e = gen.rmat(14, 16, seed=1)
    g = fb.build_csr(n, e)
    o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, snapshots=True)
    with fb.Solver(0) as s:
        s.upload(g)
        ref = {}
        for policy in (0, 1, 2):
            *_, kern1, flops1 = s.run(policy=policy, full_trace=True)
            ref[policy] = (kern1.tolist(), flops1.tolist())
    for policy in (0, 1, 2):
        kern, flops = check_oracle(n, g, ranks, policy=policy, o=o)
        assert (kern.tolist(), flops.tolist()) == ref[policy], (ranks, policy)


def test_group_skewed_graphs_hub_settings():
    rng = np.random.default_rng(91)
    for _ in range(24):
        n = int(rng.integers(300, 4000))
        k = int(rng.integers(n, 20 * n))
        u = (rng.pareto(1.2, k) * 3).astype(np.int64) % n
        v = rng.integers(0, n, k)
        g = fb.build_csr(n, np.stack([u, v], 1).astype(np.int32))
        check_oracle(n, g, int(rng.choice([2, 3, 5])), hub_slots=int(rng.choice([0, -1, 256, 1024])))


def test_group_long_rows_push_chunks():
    """Rows much longer than the push's chunk size split across ranks."""
    rng = np.random.default_rng(92)
    n = 60000
    leaves = rng.integers(0, n, n - 4)
    hub = rng.integers(0, 4, n - 4) * (n // 4)
    chain = rng.integers(0, n, (8000, 2))
    pairs = np.concatenate([np.stack([hub, leaves], 1), chain]).astype(np.int32)
    g = fb.build_csr(n, pairs)
    o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, snapshots=True)
    for ranks in (2, 4):
        for policy in (0, 2):
            check_oracle(n, g, ranks, hub_slots=0, policy=policy, o=o)
            check_oracle(n, g, ranks, hub_slots=-1, policy=policy, o=o)


def test_group_l2_rank_tier(monkeypatch):
    """The L2 rank tier (forced on a small graph) per rank."""
    monkeypatch.setenv("FSV_TIER_MIN_N", "0")
    n, e = gen.rmat(15, 16, seed=5)
    g = fb.build_csr(n, e)
    o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, snapshots=True)
    for ranks in (2, 4):
        check_oracle(n, g, ranks, o=o)


def test_group_edge_layouts_cover_every_edge_once():
    """Partitioned oriented layouts hold each undirected edge exactly once,
    and ranks with empty row ranges are allowed."""
    n, e = gen.rmat(12, 16, seed=22)
    g = fb.build_csr(n, e)
    for ranks in (2, 4, 8):
        solvers = make_group(g, ranks)
        try:
            group_run(solvers)
            total = 0
            for s in solvers:
                s.solve()
                total += int(s.stats.oriented_entries)
        finally:
            close_all(solvers)
        assert total == g.m // 2
    # tiny graph: more ranks than non-empty rows
    g = fb.build_csr(5, [(0, 1), (3, 4)])
    check_oracle(5, g, 4)


@pytest.mark.parametrize("index", [2, 3])
def test_group_baseline_configs_full_size(index):
    """BASELINE configs 2 (RMAT-22) and 3 (grid, 15 iterations) at full size,
    4 ranks: iteration count, traces, component count and label digest
    equal the golden records (made by the reference itself)."""
    rec = load_configs()[index]
    n, pairs = gen.baseline_graph(index)
    g = fb.build_csr(n, pairs)
    labels, iters, gfc, fc, snaps, kern, flops, all_labels = run_group(g, 4, snapshots=False)
    assert iters == rec["iterations"]
    assert gfc.tolist() == rec["gf_changed"] and fc.tolist() == rec["f_changed"]
    assert gen.pairs_digest(labels) == rec["labels_digest"]
    assert all(np.array_equal(x, labels) for x in all_labels)


def test_group_contract_errors():
    n, e = gen.rmat(10, 8, seed=3)
    g = fb.build_csr(n, e)
    a = fb.Solver(0)
    b = fb.Solver(0)
    try:
        a.upload(g, 0, n // 2, g.col_indices[:g.row_offsets[n // 2]])
        b.upload(g, n // 2 + 1, n, g.col_indices[g.row_offsets[n // 2 + 1]:])
        with pytest.raises(ValueError, match="cover"):
            group_run([a, b])
        with pytest.raises(ValueError, match="twice"):
            group_run([a, a])
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("ranks", [2, 4])
def test_group_sparse_delta_exchange(ranks):
    """Sparse (push) iterations exchange only the entries each rank lowered
    (k_delta_compact -> gathered lists -> k_group_delta_apply), dense ones
    min-merge the whole vector; both exchanges give the oracle's snapshots,
    and the delta exchange really ran (exchange=0) or never ran (exchange=1)."""
    n, e = gen.rmat(14, 16, seed=1)
    g = fb.build_csr(n, e)
    o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, snapshots=True)
    for policy in (0, 2):
        for exchange in (0, 1):
            solvers = make_group(g, ranks)
            try:
                labels, iters, gfc, fc, snaps, kern, flops, all_labels = group_run(
                    solvers, snapshots=True, snap_cap=64, policy=policy, exchange=exchange)
                st = solvers[0].stats
                assert iters == o.iterations and np.array_equal(snaps, o.snapshots), (policy, exchange)
                assert all(np.array_equal(x, labels) for x in all_labels)
                sparse = int(sum(1 for k in kern[1:] if k == 1))
                if exchange == 0:
                    assert st.delta_exchanges + st.dense_exchanges == iters - 1
                    assert st.delta_exchanges <= sparse and (sparse == 0 or st.delta_exchanges > 0)
                else:
                    assert st.delta_exchanges == 0 and st.dense_exchanges == iters - 1
            finally:
                close_all(solvers)
