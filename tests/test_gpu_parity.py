"""GPU parity: the sm_100a path through the C ABI against the reference's
golden vectors (tests/golden/, produced by the reference itself) and the CPU
oracle (pinned to the same vectors in test_oracle.py).

Bar: bit-exact labels, iteration count, gf_changed and f_changed traces and
every per-iteration parent vector (snapshot)."""

import numpy as np
import pytest

import oracle
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
from conftest import random_multigraph
from golden_io import load_configs, load_kats, load_suite

pytestmark = pytest.mark.gpu


def solve(solver, g, snapshots=True, hub_slots=0, batch=0):
    solver.set_hub_slots(hub_slots)
    solver.upload(g)
    return solver.run(snapshots=snapshots, snap_cap=512, batch=batch)


def check_against_oracle(solver, n, pairs, snapshots=True, hub_slots=0, batch=0):
    g = fb.build_csr(n, pairs)
    labels, iters, gfc, fc, ms, snaps = solve(solver, g, snapshots, hub_slots, batch)
    o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, snapshots=snapshots)
    assert iters == o.iterations
    assert gfc.tolist() == o.gf_changed.tolist()
    assert fc.tolist() == o.f_changed.tolist()
    assert np.array_equal(labels, o.labels)
    if snapshots:
        for k in range(iters):
            assert np.array_equal(snaps[k], o.snapshots[k]), f"snapshot {k + 1} differs"
    return g, labels, iters


@pytest.mark.parametrize("hub_slots", [0, -1, 256])
def test_golden_suite_snapshots(solver, hub_slots):
    for c in load_suite():
        g = fb.build_csr(c.n, c.edges)
        labels, iters, gfc, fc, ms, snaps = solve(solver, g, True, hub_slots)
        assert iters == c.iterations, c.name
        assert gfc.tolist() == c.gf_changed and fc.tolist() == c.f_changed, c.name
        assert np.array_equal(labels, c.labels), c.name
        assert np.array_equal(snaps, c.snapshots), c.name


def test_golden_suite_no_snapshots_batches(solver):
    # the speculative batched loop (no host sync per iteration) gives the same trace
    for c in load_suite()[::5]:
        g = fb.build_csr(c.n, c.edges)
        for batch in (1, 2, 8):
            labels, iters, gfc, fc, ms, _ = solve(solver, g, False, 0, batch)
            assert iters == c.iterations and gfc.tolist() == c.gf_changed, (c.name, batch)
            assert np.array_equal(labels, c.labels), (c.name, batch)


def test_random_multigraphs_snapshots(solver):
    rng = np.random.default_rng(71)
    for _ in range(200):
        n, pairs = random_multigraph(rng, max_n=40, density=2.5)
        check_against_oracle(solver, n, pairs)


def test_skewed_graphs_with_hub_table(solver):
    rng = np.random.default_rng(72)
    for _ in range(60):
        n = int(rng.integers(300, 3000))
        k = int(rng.integers(n, 20 * n))
        u = (rng.pareto(1.2, k) * 3).astype(np.int64) % n
        v = rng.integers(0, n, k)
        pairs = np.stack([u, v], 1).astype(np.int32)
        check_against_oracle(solver, n, pairs, snapshots=True, hub_slots=int(rng.choice([0, 256, 1024])))


def test_edge_cases(solver):
    for n, pairs in [(1, []), (2, []), (5, [(0, 0), (1, 1)]), (2, [(0, 1)]), (3, [(2, 1)]),
                     (6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)]),
                     (64, [(i, i + 1) for i in range(63)]),
                     (10, [(0, i) for i in range(1, 10)]),
                     (4099, [(i, i + 1) for i in range(4098)]),      # spans cross span/step borders
                     (3000, [(0, i) for i in range(1, 3000)])]:      # one long row
        p = np.asarray(pairs, dtype=np.int32).reshape(-1, 2)
        check_against_oracle(solver, n, p)


def test_push_long_rows_and_record_path(solver):
    """Sparse (push) iterations over very long rows (phase-B chunks) and
    dense iterations with few differing entries (record path): stars of
    thousands of leaves hung off a random forest, with and without hub slots,
    under the default and the sparse-only schedule; every snapshot equals
    the oracle's."""
    rng = np.random.default_rng(73)
    for n, centers, extra in ((20000, 3, 2000), (120000, 8, 30000), (70000, 1, 0)):
        leaves = rng.integers(0, n, n - centers)
        hub = rng.integers(0, centers, n - centers)
        star = np.stack([hub * (n // max(centers, 1)), leaves], 1)
        chain = np.stack([rng.integers(0, n, extra), rng.integers(0, n, extra)], 1)
        pairs = np.concatenate([star, chain]).astype(np.int32)
        g = fb.build_csr(n, pairs)
        o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, snapshots=True)
        for hub_slots in (0, -1):
            solver.set_hub_slots(hub_slots)
            solver.upload(g)
            for policy in (0, 2):
                labels, iters, gfc, fc, ms, snaps = solver.run(snapshots=True, snap_cap=64, policy=policy)
                assert iters == o.iterations and gfc.tolist() == o.gf_changed.tolist(), (n, hub_slots, policy)
                assert np.array_equal(snaps, o.snapshots), (n, hub_slots, policy)
    solver.set_hub_slots(0)


def test_empty_graph_runs_one_iteration():
    r = fb.fastsv_la(fb.build_csr(0, []))
    assert r.iterations == 1 and r.labeling.component_count == 0


def test_public_api_matches_reference_kats():
    k = load_kats()
    r = fb.fastsv_la(fb.build_csr(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)]))
    assert r.labeling.labels.tolist() == k["two_triangles"]["labels"]
    assert r.labeling.labels.dtype == np.int64
    r = fb.fastsv(fb.build_csr(10, [(0, i) for i in range(1, 10)]))
    assert r.iterations == k["star10"]["iterations"]
    r = fb.fastsv_la(fb.build_csr(64, [(i, i + 1) for i in range(63)]), record_snapshots=True)
    assert r.iterations == k["path64_fastsv"]["iterations"] == len(r.snapshots)
    assert all(not s.flags.writeable for s in r.snapshots)
    assert r.trace[-1].gf_changed == 0 and all(t.gf_changed > 0 for t in r.trace[:-1])
    assert r.total_elapsed > 0


def test_reference_style_int64_csr_is_accepted():
    # a CsrGraph exactly like svcc's (int64 columns) goes through fsv_upload_csr64
    n, e = gen.rmat(10, 8, seed=4)
    g = fb.build_csr(n, e)
    g64 = fb.CsrGraph(n=n, row_offsets=g.row_offsets, col_indices=g.col_indices.astype(np.int64))
    a = fb.fastsv_la(g)
    b = fb.fastsv_la(g64)
    assert a.iterations == b.iterations and np.array_equal(a.labeling.labels, b.labeling.labels)


def test_connected_components_edge_list():
    n, e = gen.forest(500, 1, 64, 2, seed=8)
    labels = fb.connected_components(n, e)
    assert np.array_equal(labels, oracle.uf_labels(n, e).astype(np.int64))


def test_upload_rejects_out_of_range_columns(solver):
    off = np.array([0, 1, 2], dtype=np.int64)
    cols = np.array([1, 7], dtype=np.int32)
    with pytest.raises(fb.InputError, match="out of range for n=2"):
        solver.upload(fb.CsrGraph(n=2, row_offsets=off, col_indices=cols))


@pytest.mark.parametrize("index", [1, 2, 3, 4])
def test_baseline_config_full_size(solver, index):
    rec = load_configs()[index]
    n, pairs = gen.baseline_graph(index)
    assert gen.pairs_digest(pairs) == rec["pairs_digest"]
    g = fb.build_csr(n, pairs)
    solver.set_hub_slots(0)
    solver.upload(g)
    labels, iters, gfc, fc, ms, _ = solver.run()
    assert iters == rec["iterations"]
    assert gfc.tolist() == rec["gf_changed"] and fc.tolist() == rec["f_changed"]
    assert gen.pairs_digest(labels) == rec["labels_digest"]
    assert solver.stats.component_count == rec["component_count"]
    if index == 1:
        assert np.array_equal(labels, oracle.uf_labels(n, pairs))


@pytest.mark.parametrize("hub_slots", [55296, 24576, 4096])
def test_config2_hub_table_sizes(solver, hub_slots):
    """The hub table size is a performance knob (default 47,104 slots: 192 KB of
    shared memory; 55,296 is the largest table, 24,576 the rank-tier default):
    the result does not depend on it."""
    rec = load_configs()[2]
    n, pairs = gen.baseline_graph(2)
    g = fb.build_csr(n, pairs)
    solver.set_hub_slots(hub_slots)
    solver.upload(g)
    labels, iters, gfc, fc, ms, _ = solver.run()
    solver.set_hub_slots(0)
    assert solver.stats.hub_slots == hub_slots
    assert iters == rec["iterations"]
    assert gfc.tolist() == rec["gf_changed"] and fc.tolist() == rec["f_changed"]
    assert gen.pairs_digest(labels) == rec["labels_digest"]


def test_default_hub_table_keeps_l1(solver):
    """Default table: 47,104 slots (with the hot accumulators 192 KB, below the
    carve-out step that halves the random-gather rate)."""
    n, pairs = gen.baseline_graph(2)
    solver.set_hub_slots(0)
    solver.upload(fb.build_csr(n, pairs))
    solver.solve()
    assert solver.stats.hub_slots == 47104


@pytest.mark.parametrize("index", [1, 2])
def test_minority_sweep_on_and_off(solver, index):
    """The minority sweep of late dense iterations (fsv_set_minority_sweep)
    visits only the edges at vertices outside the majority grandparent; the
    trace and the labels are the reference's with it and without it."""
    rec = load_configs()[index]
    n, pairs = gen.baseline_graph(index)
    solver.set_hub_slots(0)
    solver.upload(fb.build_csr(n, pairs))
    try:
        for on in (False, True):
            solver.set_minority_sweep(on)
            for batch in (0, 1):      # graph loop and host loop
                labels, iters, gfc, fc, ms, _ = solver.run(batch=batch)
                assert iters == rec["iterations"], (on, batch)
                assert gfc.tolist() == rec["gf_changed"] and fc.tolist() == rec["f_changed"], (on, batch)
                assert gen.pairs_digest(labels) == rec["labels_digest"], (on, batch)
                if index == 2:    # RMAT-22: the third iteration is the minority one
                    assert solver.stats.minority_iterations == (1 if on else 0), (on, batch)
    finally:
        solver.set_minority_sweep(True)


def test_minority_sweep_snapshots_on_skewed_graphs(solver):
    """Every per-iteration parent vector with the minority sweep on (RMAT and
    star-heavy graphs with a hub table, where a giant component dominates
    from the third iteration)."""
    took = 0
    for scale, ef, seed in ((14, 16, 3), (15, 8, 4), (16, 16, 5), (15, 16, 6)):
        n, pairs = gen.rmat(scale, ef, seed=seed)
        if seed == 6:   # n % 4 != 0: the scalar tail group of the minority list
            pairs = np.concatenate([pairs, np.array([[n, n + 1], [n + 2, 5], [n + 1, 7]], dtype=np.int32)])
            n += 3
        g = fb.build_csr(n, pairs)
        o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, snapshots=True)
        for hub_slots in (0, 1024):
            solver.set_hub_slots(hub_slots)
            solver.upload(g)
            for policy in (3, 1):     # auto and dense-only schedules
                labels, iters, gfc, fc, ms, snaps = solver.run(snapshots=True, snap_cap=64, policy=policy)
                assert iters == o.iterations and gfc.tolist() == o.gf_changed.tolist(), (scale, hub_slots, policy)
                assert np.array_equal(snaps, o.snapshots), (scale, hub_slots, policy)
            solver.solve()
            took += solver.stats.minority_iterations
    solver.set_hub_slots(0)
    assert took > 0       # (the sweep did run on these graphs)


POLICY = {"auto": (3, 0.1), "auto_t1": (3, 1.0), "auto_t05": (3, 0.5), "sparse_only": (2, 0.1),
          "dense_only": (1, 0.1)}


def test_product_schedule_matches_reference_trace(solver):
    """Same per-iteration product choice (dense pull / sparse push) and the
    same flops as the reference's IterationTrace under five DriverConfigs;
    snapshots stay identical to the golden ones under every schedule."""
    from golden_io import load_driver_traces
    traces = load_driver_traces()
    suite = {c.name: c for c in load_suite()}
    checked = 0
    for (cfg, name), (kinds, flops) in traces.items():
        c = suite[name]
        g = fb.build_csr(c.n, c.edges)
        solver.set_hub_slots(0)
        solver.upload(g)
        policy, thr = POLICY[cfg]
        labels, iters, gfc, fc, ms, snaps, kern, fl = solver.run(
            snapshots=True, snap_cap=512, policy=policy, threshold=thr, full_trace=True)
        assert iters == c.iterations and np.array_equal(snaps, c.snapshots), (cfg, name)
        assert kern.tolist() == kinds, (cfg, name)
        assert fl.tolist() == flops, (cfg, name)
        checked += 1
    assert checked >= 400


def test_public_api_trace_fields_match_reference():
    g = fb.build_csr(64, [(i, i + 1) for i in range(63)])
    r = fb.fastsv_la(g, fb.DriverConfig(sparse_threshold=1.0))
    assert r.trace[0].kernel == "dense"                      # test_driver.py:110-114
    assert all(t.kernel == "sparse" for t in r.trace[1:])
    r = fb.fastsv_la(g, fb.DriverConfig(force_kernel="sparse_only"))
    assert r.trace[0].kernel == "sparse" and r.trace[0].flops == g.m   # test_driver.py:117-121
    r = fb.fastsv_la(g, fb.DriverConfig(force_kernel="dense_only"))
    assert all(t.kernel == "dense" and t.flops == g.m for t in r.trace)  # test_driver.py:124-127


def test_single_rank_nccl_path_matches():
    """The multi-GPU code path (NCCL allreduce-min every iteration, f1
    assembled by allreduce at upload) with one rank: identical results."""
    n, e = gen.rmat(13, 16, seed=21)
    g = fb.build_csr(n, e)
    o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices)
    with fb.Solver(0) as s:
        s.attach_nccl(fb.Solver.nccl_unique_id(), 1, 0)
        s.upload(g)
        labels, iters, gfc, fc, ms, _ = s.run()
        assert iters == o.iterations and gfc.tolist() == o.gf_changed.tolist()
        assert np.array_equal(labels, o.labels)
        # the collective captured into the CUDA-graph loop (one host sync per
        # solve) when NCCL accepts capture there, else the host loop
        print("nccl single-rank host_syncs:", s.stats.host_syncs)
        for batch in (1, 3):
            labels2, iters2, gfc2, *_ = s.run(batch=batch)
            assert iters2 == iters and np.array_equal(labels2, labels)


def test_row_partition_upload_two_contexts_emulate_ranks():
    """Two contexts on one GPU, each owning half the rows, run WITHOUT a
    communicator cannot merge; instead check the partitioned layout covers
    every edge exactly once: the union of the two ranks' oriented entries
    equals the single-rank layout size."""
    n, e = gen.rmat(12, 16, seed=22)
    g = fb.build_csr(n, e)
    import bench
    sizes = []
    for r in range(2):
        lo, hi = bench.row_partition(g.row_offsets, 2, r)
        with fb.Solver(0) as s:
            s.upload(g, lo, hi, g.col_indices[g.row_offsets[lo]:g.row_offsets[hi]])
            sizes.append(int(s.solve().oriented_entries))
    with fb.Solver(0) as s:
        s.upload(g)
        total = int(s.solve().oriented_entries)
    assert sum(sizes) == total == g.m // 2


def test_graph_loop_and_host_loop_agree(solver):
    """The CUDA-graph conditional-WHILE loop (default) and the host-driven
    speculative batches produce identical traces; per-iteration device times
    come from %globaltimer stamps."""
    n, e = gen.rmat(14, 16, seed=31)
    g = fb.build_csr(n, e)
    solver.set_hub_slots(0)
    solver.upload(g)
    a = solver.run()                  # graph mode
    st_graph = (int(solver.stats.host_syncs), int(solver.stats.kernel_launches))
    b = solver.run(batch=2)           # host loop
    assert a[1] == b[1] and a[2].tolist() == b[2].tolist() and np.array_equal(a[0], b[0])
    assert st_graph[0] == 1
    assert all(ms > 0 for ms in a[4])


def test_rank_tier_path(solver, monkeypatch):
    """The L2 rank tier (degree-ranked compact gf beyond the shared-memory
    slots; on by default only when the vectors overflow L2) forced on small
    skewed graphs with a small shared-memory table: identical results."""
    monkeypatch.setenv("FSV_TIER_MIN_N", "0")
    for seed, scale in ((41, 12), (42, 13), (43, 14)):
        n, e = gen.rmat(scale, 16, seed=seed)
        g = fb.build_csr(n, e)
        o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, snapshots=True)
        solver.set_hub_slots(256)
        solver.upload(g)
        st = solver.solve()
        assert st.hub_slots > 256           # the tier is in use
        for policy in (0, 1):
            labels, iters, gfc, fc, ms, snaps = solver.run(snapshots=True, snap_cap=64, policy=policy)
            assert iters == o.iterations and gfc.tolist() == o.gf_changed.tolist()
            assert np.array_equal(snaps, o.snapshots)
    solver.set_hub_slots(0)


# ---- device CSR build from edge lists (fsv_upload_edges, graph.py:55-97) ----

def test_device_csr_build_matches_reference_suite(solver):
    """fsv_upload_edges builds exactly svcc.build_csr's arrays (reference-made
    digests) and the solve on that CSR matches the reference's golden run."""
    from golden_io import csr_digest, load_csr_digests
    gold = load_csr_digests()["suite"]
    solver.set_hub_slots(0)
    for i, c in enumerate(load_suite()):
        pairs = c.edges if i % 2 else c.edges.astype(np.int64)    # both id widths
        solver.upload_edges(c.n, pairs)
        g = solver.csr()
        assert g.m == c.m_dir, c.name
        assert csr_digest(g.row_offsets, g.col_indices) == gold[c.name]["digest"], c.name
        labels, iters, gfc, fc, ms, snaps = solver.run(snapshots=True, snap_cap=512)
        assert iters == c.iterations and gfc.tolist() == c.gf_changed, c.name
        assert np.array_equal(labels, c.labels) and np.array_equal(snaps, c.snapshots), c.name


@pytest.mark.parametrize("index", [1, 2, 3, 4])
def test_device_csr_build_baseline_configs(solver, index):
    """Full-size configs: the device-built CSR equals the reference's (digest,
    configs 1 and 3) or the host builder's arrays (configs 2 and 4, whose
    reference build takes minutes), and the solve reproduces the golden run."""
    from golden_io import csr_digest, load_csr_digests
    rec = load_configs()[index]
    n, pairs = gen.baseline_graph(index)
    solver.set_hub_slots(0)
    solver.upload_edges(n, pairs)
    g = solver.csr()
    assert g.m == rec["m_dir"]
    gold = load_csr_digests()["configs"].get(str(index))
    if gold is not None:
        assert csr_digest(g.row_offsets, g.col_indices) == gold["digest"]
    else:
        h = fb.build_csr(n, pairs)
        assert np.array_equal(g.row_offsets, h.row_offsets)
        assert np.array_equal(g.col_indices, h.col_indices)
    labels, iters, gfc, fc, ms, _ = solver.run()
    assert iters == rec["iterations"] and gfc.tolist() == rec["gf_changed"]
    assert gen.pairs_digest(labels) == rec["labels_digest"]


def test_device_csr_build_edge_cases(solver):
    solver.set_hub_slots(0)
    cases = [
        (0, np.zeros((0, 2), np.int32)),
        (1, np.zeros((0, 2), np.int32)),
        (1, np.array([[0, 0]], np.int32)),                      # self-loop only
        (5, np.array([[3, 3], [1, 1]], np.int64)),
        (6, np.array([[5, 0], [0, 5], [5, 0], [2, 2], [4, 1]], np.int32)),
        (3, [(0, 1), (1, 2)]),                                    # list input
        (2 ** 20, np.array([[2 ** 20 - 1, 0], [7, 2 ** 19]], np.int64)),
    ]
    for n, e in cases:
        solver.upload_edges(n, e)
        g = solver.csr()
        h = fb.build_csr(n, e)
        assert np.array_equal(g.row_offsets, h.row_offsets), (n, e)
        assert np.array_equal(g.col_indices, h.col_indices), (n, e)
        if n:
            labels, *_ = solver.run()
            assert np.array_equal(labels, oracle.uf_labels(n, np.asarray(e, np.int64).reshape(-1, 2))), (n, e)


def test_device_csr_build_errors(solver):
    # the first offending pair in input order, with the reference's message
    with pytest.raises(fb.InputError, match=r"edge \(5, -1\) out of range for n=10"):
        solver.upload_edges(10, np.array([[0, 1], [5, -1], [7, 100]], np.int64))
    with pytest.raises(fb.InputError, match=r"edge \(7, 10\) out of range for n=10"):
        solver.upload_edges(10, np.array([[0, 1], [7, 10], [3, -4]], np.int32))
    with pytest.raises(fb.InputError, match="vertex count must be non-negative"):
        solver.upload_edges(-1, [])
    with pytest.raises(fb.InputError, match=r"edges must be \(u, v\) pairs"):
        solver.upload_edges(4, np.zeros((2, 3), np.int64))
    # a failed upload leaves the context usable
    solver.upload_edges(4, [(0, 1), (2, 3)])
    labels, *_ = solver.run()
    assert labels.tolist() == [0, 0, 2, 2]


def test_device_csr_build_row_ranges():
    """Two contexts each build the CSR and keep half the rows: every
    undirected edge is oriented by exactly one of them, and each keeps the
    reference's columns of its rows."""
    n, e = gen.rmat(12, 16, seed=23)
    h = fb.build_csr(n, e)
    import bench
    sizes = []
    for r in range(2):
        lo, hi = bench.row_partition(h.row_offsets, 2, r)
        with fb.Solver(0) as s:
            s.upload_edges(n, e, lo, hi)
            g = s.csr()
            assert np.array_equal(g.row_offsets, h.row_offsets)
            assert np.array_equal(g.col_indices, h.col_indices[h.row_offsets[lo]:h.row_offsets[hi]])
            sizes.append(int(s.solve().oriented_entries))
    assert sum(sizes) == h.m // 2


# ---- hooking variants and simplified_sv (fsv_config.hooking) ----------------

def _snap_digest(snaps):
    import hashlib
    h = hashlib.sha256()
    for s in snaps:
        h.update(np.ascontiguousarray(s, dtype="<i8").tobytes())
    return h.hexdigest()[:16]


def test_hooking_variants_match_reference_traces(solver):
    """Every HookingConfig (16 flag sets) and simplified_sv on every golden
    graph: iteration count, gf_changed/f_changed traces and every committed
    parent vector (snapshot digest) equal the reference's own runs."""
    from golden_io import load_variants, variant_graphs
    from paper_1910_05971_b200.driver import HOOKING_SET
    runs, extra = load_variants()
    graphs = variant_graphs()
    for name, digest in extra.items():
        assert gen.pairs_digest(graphs[name][1]) == digest, name
    solver.set_hub_slots(0)
    current = None
    for name, code, iters, gfc, fc, digest in runs:
        if name != current:
            n, e = graphs[name]
            solver.upload(fb.build_csr(n, e))
            current = name
        hooking = HOOKING_SET if code == 16 else HOOKING_SET | code
        labels, k, g2, f2, ms, snaps, kern, flops = solver.run(snapshots=True, snap_cap=64, hooking=hooking,
                                                               full_trace=True)
        assert (k, g2.tolist(), f2.tolist()) == (iters, gfc, fc), (name, code)
        assert _snap_digest(snaps) == digest, (name, code)
        assert all(x == 2 for x in kern) and all(x == 0 for x in flops)


def test_public_variant_api():
    """fastsv(g, HookingConfig(...)), simplified_sv and the sv1..sv5 ablation
    through the public API: RunResult shape of the reference."""
    n, e = gen.rmat(11, 8, seed=41)
    g = fb.build_csr(n, e)
    uf = oracle.uf_labels(n, e).astype(np.int64)
    r = fb.simplified_sv(g, record_snapshots=True)
    assert np.array_equal(r.labeling.labels, uf) and len(r.snapshots) == r.iterations
    assert all(t.kernel == "none" and t.flops == 0 for t in r.trace)
    r3 = fb.fastsv(g, fb.sv_level_config(3))
    assert np.array_equal(r3.labeling.labels, uf)
    suite = fb.ablation_suite(g)
    assert [s[0] for s in suite] == ["sv1", "sv2", "sv3", "sv4", "sv5"]
    assert suite[4][1] == fb.fastsv(g).iterations


def test_bounds_checked_build_runs_clean():
    """The -DFSV_CHECKS build (libfastsv_checked.so: every vertex-array load
    and min-reduction of a solve checked against the registered buffers, trap
    on a miss) solves the golden suite sample, skewed graphs with hub slots,
    sparse-only schedules and a row partition without a trap, bit-exactly.
    Run in a subprocess: a trap poisons the CUDA context."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    lib = root / "paper_1910_05971_b200" / "libfastsv_checked.so"
    if not lib.exists():
        pytest.skip("libfastsv_checked.so not built")
    env = dict(os.environ, FSV_LIB=str(lib))
    r = subprocess.run([sys.executable, str(root / "tools" / "sanitize_run.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "(single context) done, mismatches: 0" in r.stdout, r.stdout[-2000:]
    assert "groups) done, mismatches: 0" in r.stdout, r.stdout[-2000:]


def test_graph_reuse_across_uploads_of_the_same_shape(solver):
    """Re-uploads that keep every captured buffer and size keep the
    instantiated iteration graph: alternating a graph and a relabelled copy
    of it (same sizes, different contents) must still give each one's own
    oracle result."""
    n, e = gen.rmat(14, 16, seed=91)
    perm = np.random.default_rng(92).permutation(n).astype(np.int32)
    graphs = [fb.build_csr(n, e), fb.build_csr(n, perm[e])]
    oracles = [oracle.fastsv_csr(n, g.row_offsets, g.col_indices) for g in graphs]
    solver.set_hub_slots(0)
    for rep in range(3):
        for g, o in zip(graphs, oracles):
            solver.upload(g)
            labels, iters, gfc, fc, ms, _ = solver.run()
            assert iters == o.iterations and gfc.tolist() == o.gf_changed.tolist(), rep
            assert np.array_equal(labels, o.labels), rep


def test_device_labeling_matches_reference_labeling(solver):
    """Labeling built on the device (fsv_get_labeling: int64 labels, count,
    sizes) equals the reference's labeling_from_parents (graph.py:109-125)
    on the golden suite and on skewed/forest graphs."""
    graphs = [(c.n, c.edges) for c in load_suite()[::3]]
    graphs += [gen.rmat(14, 16, seed=9), gen.forest(3000, 1, 64, 2, seed=2), (1, []), (7, [])]
    for n, e in graphs:
        g = fb.build_csr(n, e)
        solver.set_hub_slots(0)
        solver.upload(g)
        solver.solve()
        lab = solver.labeling()
        ref = fb.labeling_from_parents(solver.labels().astype(np.int64))
        assert lab.labels.dtype == np.int64 and np.array_equal(lab.labels, ref.labels)
        assert lab.component_count == ref.component_count
        assert lab.sizes == ref.sizes and dict(lab.sizes.items()) == ref.sizes
        assert sum(lab.sizes.values()) == n
        if n:
            r = int(lab.labels[0])
            assert lab.sizes[r] == ref.sizes[r]
    r = fb.fastsv_la(fb.build_csr(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)]))
    assert r.labeling.sizes == {0: 3, 3: 3} and r.labeling.component_count == 2


def test_config5_full_size_matches_oracle_record():
    """BASELINE config 5 (RMAT-27: 2^31 pairs, ~4.2e9 directed entries, int64
    offsets) on one B200: the edge list goes up, the CSR is built on the
    device (fsv_upload_edges), and the solve must reproduce the golden record
    of the C oracle (tests/golden/make_config5_golden.py; the Python
    reference is infeasible at this size): iteration count,
    gf_changed / f_changed per iteration, component count, label digest."""
    rec = load_configs().get(5)
    if rec is None:
        pytest.skip("tests/golden/configs.json has no config 5 record yet")
    n, pairs = gen.baseline_graph(5)
    assert gen.pairs_digest(pairs) == rec["pairs_digest"]
    with fb.Solver(0) as solver:       # its own context: ~60 GB of device memory, freed after
        solver.upload_edges(n, pairs)
        del pairs
        assert solver.m == rec["m_dir"]
        labels, iters, gfc, fc, ms, _ = solver.run()
        assert iters == rec["iterations"]
        assert gfc.tolist() == rec["gf_changed"] and fc.tolist() == rec["f_changed"]
        assert solver.stats.component_count == rec["component_count"]
        assert gen.pairs_digest(labels) == rec["labels_digest"] == rec["uf_labels_digest"]


def test_repeated_solves_are_deterministic(solver):
    """Functional race detector: the BSP schedule makes every
    solve's trace identical, whatever the interleaving of the atomics. 40
    solves each of config 3 (15 iterations: the config whose iteration count
    a rejected round-1 kernel variant once got wrong) and config 2 (hub
    table, record path, push), alternating the CUDA-graph loop and the
    host-batched loop, must all reproduce the reference's golden record."""
    for index in (3, 2):
        rec = load_configs()[index]
        n, pairs = gen.baseline_graph(index)
        g = fb.build_csr(n, pairs)
        solver.set_hub_slots(0)
        solver.upload(g)
        for i in range(40):
            st = solver.solve(batch=0 if i % 2 == 0 else 3)
            assert st.iterations == rec["iterations"], (index, i)
            gfc, fc, _ = solver.trace()
            assert gfc.tolist() == rec["gf_changed"] and fc.tolist() == rec["f_changed"], (index, i)
            if i % 8 == 0:
                assert gen.pairs_digest(solver.labels()) == rec["labels_digest"], (index, i)


def test_column_tiled_layout_matches_golden(solver, monkeypatch):
    """Column-range tiling of the oriented layout (k_tile_pass: layouts
    without hubs or huge rows, each row split into per-tile segments) forced
    on small graphs by a tiny tile width: every per-iteration parent vector
    of the golden suite, random multigraphs and forests equals the
    reference's / the oracle's (configs 3 and 4 take the tiled layout by
    default and are checked at full size by test_baseline_config_full_size)."""
    rng = np.random.default_rng(93)
    for width, chunks in (("7", None), ("64", "3"), ("1000", None)):
        monkeypatch.setenv("FSV_TILE_W", width)
        if chunks:   # chunked host upload: encode per chunk, tiles compacted over all rows after
            monkeypatch.setenv("FSV_UPLOAD_CHUNKS", chunks)
        else:
            monkeypatch.delenv("FSV_UPLOAD_CHUNKS", raising=False)
        for c in load_suite()[::4]:
            g = fb.build_csr(c.n, c.edges)
            labels, iters, gfc, fc, ms, snaps = solve(solver, g, True, -1)
            assert iters == c.iterations and gfc.tolist() == c.gf_changed, (width, c.name)
            assert np.array_equal(snaps, c.snapshots), (width, c.name)
        for _ in range(20):
            n, pairs = random_multigraph(rng, max_n=300, density=1.5)
            check_against_oracle(solver, n, pairs, hub_slots=-1)
        n, e = gen.forest(400, 1, 64, 2, seed=int(rng.integers(1 << 30)))
        check_against_oracle(solver, n, e, hub_slots=-1)
        # with a hub table (hub-coded columns go to the first tile) and rows
        # long enough for the huge-row pieces
        for _ in range(4):
            n = int(rng.integers(2000, 6000))
            k = int(rng.integers(4 * n, 20 * n))
            u = (rng.pareto(1.1, k) * 2).astype(np.int64) % n
            v = rng.integers(0, n, k)
            check_against_oracle(solver, n, np.stack([u, v], 1).astype(np.int32), hub_slots=256)
        n, e = gen.rmat(14, 16, seed=int(rng.integers(1 << 30)))
        check_against_oracle(solver, n, e, hub_slots=0)
        monkeypatch.setenv("FSV_TIER_MIN_N", "0")   # and the L2 rank tier
        check_against_oracle(solver, n, e, hub_slots=0)
        monkeypatch.delenv("FSV_TIER_MIN_N")
    monkeypatch.delenv("FSV_TILE_W")
    monkeypatch.delenv("FSV_UPLOAD_CHUNKS", raising=False)
    solver.set_hub_slots(0)
