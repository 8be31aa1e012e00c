"""Host-side logic of the drop-in: graph building, labels, configs, errors,
generators. No GPU needed."""

import numpy as np
import pytest

import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import errors, generators as gen
from golden_io import load_suite


def test_build_csr_semantics():
    # symmetrise, dedup, drop self-loops, sorted rows (graph.py:55-97)
    g = fb.build_csr(4, [(1, 0), (0, 1), (2, 2), (3, 1), (1, 3)])
    assert g.row_offsets.tolist() == [0, 1, 3, 3, 4]
    assert g.col_indices.tolist() == [1, 0, 3, 1]
    assert g.m == 4 and g.degrees.tolist() == [1, 2, 0, 1]
    assert g.row_ids.tolist() == [0, 1, 1, 3]
    assert not g.row_offsets.flags.writeable and not g.col_indices.flags.writeable
    assert g.neighbors(1).tolist() == [0, 3]


def test_build_csr_matches_reference_sizes():
    for c in load_suite():
        assert fb.build_csr(c.n, c.edges).m == c.m_dir, c.name


def test_build_csr_errors():
    with pytest.raises(fb.InputError, match=r"\(1, 3\).*n=3"):
        fb.build_csr(3, [(0, 1), (1, 3)])
    with pytest.raises(fb.InputError):
        fb.build_csr(-1, [])
    with pytest.raises(fb.InputError):
        fb.build_csr(3, np.zeros((2, 3), dtype=np.int64))
    g = fb.build_csr(0, [])
    assert g.n == 0 and g.m == 0
    g = fb.build_csr(5, np.zeros((0, 2), dtype=np.int32))
    assert g.row_offsets.tolist() == [0] * 6


def test_int32_and_int64_inputs_agree():
    rng = np.random.default_rng(3)
    e = rng.integers(0, 300, (2000, 2))
    a = fb.build_csr(300, e)
    b = fb.build_csr(300, e.astype(np.int32))
    assert np.array_equal(a.row_offsets, b.row_offsets) and np.array_equal(a.col_indices, b.col_indices)


def test_labeling_from_parents():
    lab = fb.labeling_from_parents(np.array([0, 0, 2, 2, 0]))
    assert lab.component_count == 2 and lab.sizes == {0: 3, 2: 2}
    assert lab.labels.dtype == np.int64
    with pytest.raises(fb.InvariantError):
        fb.labeling_from_parents(np.array([0, 0, 1]))


def test_driver_config_and_choose_kernel():
    # test_driver.py:29-49
    cfg = fb.DriverConfig(sparse_threshold=0.1)
    assert fb.choose_kernel(5, 100, cfg) == "sparse"
    assert fb.choose_kernel(10, 100, cfg) == "dense"
    assert fb.choose_kernel(100, 100, cfg) == "dense"
    zero = fb.DriverConfig(sparse_threshold=0.0)
    assert fb.choose_kernel(0, 100, zero) == "dense"
    assert fb.choose_kernel(100, 100, fb.DriverConfig(force_kernel="sparse_only")) == "sparse"
    assert fb.choose_kernel(0, 100, fb.DriverConfig(force_kernel="dense_only")) == "dense"
    for bad in (dict(sparse_threshold=-0.1), dict(sparse_threshold=1.5),
                dict(force_kernel="fast_please"), dict(workers=0), dict(batch=-1)):
        with pytest.raises(ValueError):
            fb.DriverConfig(**bad)


def test_hooking_variant_codes():
    """HookingConfig -> fsv_config.hooking (include/fastsv.h) and the sv1..sv5
    ladder of algorithms.py:170-181."""
    from paper_1910_05971_b200.driver import HOOKING_SET, hooking_code
    assert [hooking_code(fb.sv_level_config(k)) for k in range(1, 6)] == \
        [HOOKING_SET, HOOKING_SET | 1, HOOKING_SET | 3, HOOKING_SET | 7, HOOKING_SET | 15]
    assert hooking_code(fb.HookingConfig()) == HOOKING_SET | 15
    with pytest.raises(ValueError, match="sv level must be 1..5"):
        fb.sv_level_config(0)


@pytest.mark.skipif(fb.device_count() > 0, reason="checks the no-GPU behaviour")
def test_variants_fail_loudly_without_a_gpu():
    g = fb.build_csr(3, [(0, 1)])
    with pytest.raises(fb.DeviceError):
        fb.fastsv(g, fb.HookingConfig(stochastic_hooking=False))
    with pytest.raises(fb.DeviceError):
        fb.simplified_sv(g)


def test_status_mapping():
    errors.raise_for_status(0, "")
    for code, exc in ((1, fb.InputError), (2, ValueError), (3, fb.InvariantError), (4, fb.DeviceError)):
        with pytest.raises(exc, match="boom"):
            errors.raise_for_status(code, "boom")


def test_generators_deterministic_and_pinned():
    n, a = gen.rmat(10, 16, seed=7)
    _, b = gen.rmat(10, 16, seed=7)
    _, c = gen.rmat(10, 16, seed=8)
    assert n == 1024 and a.shape == (16384, 2) and a.dtype == np.int32
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert a.min() >= 0 and a.max() < n
    n, e = gen.grid(10, 12, 0.0, seed=1, permute=False)
    assert n == 120 and e.shape[0] == 10 * 11 + 9 * 12
    n, e = gen.grid(10, 12, 1.0, seed=1)
    assert e.shape[0] == 0
    n, e = gen.forest(100, 1, 64, 2, seed=3)
    assert e.shape[0] == n - 100 + 200
    # forest has exactly `trees` components
    import oracle
    assert len(np.unique(oracle.uf_labels(n, e))) == 100


def test_permutation_is_bijection():
    import ctypes
    from paper_1910_05971_b200._native import graphgen_lib
    p = np.empty(1000, dtype=np.int32)
    assert graphgen_lib().fsvg_permutation(1000, 11, p.ctypes.data) == 0
    assert sorted(p.tolist()) == list(range(1000))


def test_build_csr_matches_reference_arrays():
    """The host CSR builder reproduces svcc.build_csr's arrays exactly
    (digests made by the reference itself, tests/golden/make_csr_golden.py)."""
    from golden_io import csr_digest, load_csr_digests
    gold = load_csr_digests()["suite"]
    for c in load_suite():
        g = fb.build_csr(c.n, c.edges)
        assert csr_digest(g.row_offsets, g.col_indices) == gold[c.name]["digest"], c.name


@pytest.mark.parametrize("index", [1, 2, 3, 4])
def test_build_csr_matches_reference_arrays_baseline_configs(index):
    """BASELINE configs 1-4 at full size: the host builder's CSR equals the
    one svcc.build_csr produced (digests made by the reference itself,
    tests/golden/make_csr_golden.py --configs; 244 s for config 2 there)."""
    from golden_io import csr_digest, load_csr_digests
    rec = load_csr_digests()["configs"][str(index)]
    n, pairs = gen.baseline_graph(index)
    assert gen.pairs_digest(pairs) == rec["pairs_digest"]
    g = fb.build_csr(n, pairs)
    assert g.m == rec["m_dir"]
    assert csr_digest(g.row_offsets, g.col_indices) == rec["digest"]
