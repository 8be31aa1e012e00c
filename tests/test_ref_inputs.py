"""The reference arm's numpy inputs (baseline/ref_inputs.py) are the same
graphs as the repo's C++ generators and CSR builder produce: same pairs,
same symmetric CSR (svcc.build_csr semantics, pinned to the reference's own
arrays in tests/golden/csr_digests.json through the C++ builder)."""

import numpy as np
import pytest

import paper_1910_05971_b200 as fb
from baseline import ref_inputs as R
from paper_1910_05971_b200 import generators as gen


@pytest.mark.parametrize("case", ["rmat", "grid", "forest", "gnm"])
def test_generators_match_cpp(case):
    if case == "rmat":
        a, b = R.rmat(13, 16, seed=3), gen.rmat(13, 16, seed=3)
    elif case == "grid":
        a, b = R.grid(257, 301, 0.4, seed=4), gen.grid(257, 301, 0.4, seed=4)
    elif case == "forest":
        a, b = R.forest(2000, 1, 64, 2, seed=5), gen.forest(2000, 1, 64, 2, seed=5)
    else:
        a, b = R.baseline_graph(1), gen.baseline_graph(1)
    assert a[0] == b[0] and np.array_equal(a[1], b[1])
    off, cols = R.csr(a[0], a[1])
    g = fb.build_csr(b[0], b[1])
    assert np.array_equal(off, g.row_offsets) and np.array_equal(cols, g.col_indices)
    assert off.dtype == np.int64 and cols.dtype == np.int64


def test_csr_semantics_small():
    off, cols = R.csr(6, np.array([[0, 1], [1, 0], [2, 2], [5, 3], [0, 1]], dtype=np.int32))
    assert off.tolist() == [0, 1, 2, 2, 3, 3, 4]
    assert cols.tolist() == [1, 0, 5, 3]
