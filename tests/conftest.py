"""Shared fixtures. ``gpu``-marked tests need a B200 and the built CUDA
library; everything else runs on the CPU (oracle vs golden vectors, host
logic, ABI exports, multi-rank schedule over gloo)."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device and libfastsv.so")
    config.addinivalue_line("markers", "slow: full BASELINE-size case (minutes of CPU oracle time)")


@pytest.fixture(scope="session")
def golden_suite():
    """Reference-produced golden vectors (tests/golden/make_golden.py)."""
    path = GOLDEN / "suite.npz"
    data = np.load(path, allow_pickle=False)
    return data


def random_multigraph(rng, max_n=16, density=2.0):
    """(n, raw int32 pairs) with self-loops and duplicates on purpose
    (the reference's conftest.random_graph shape, tests/conftest.py:62-72)."""
    n = int(rng.integers(1, max_n + 1))
    k = int(rng.integers(0, max(1, int(n * density)) + 1))
    return n, rng.integers(0, n, (k, 2)).astype(np.int32)


@pytest.fixture(scope="session")
def solver():
    from paper_1910_05971_b200 import Solver
    s = Solver(0)
    yield s
    s.close()
