"""The C-ABI boundary: both libraries load and export every symbol their
headers declare; status codes, error strings and the no-CPU-fallback rule.
No compute call needs a GPU here."""

import re
from pathlib import Path

import pytest

import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import _native

ROOT = Path(__file__).resolve().parent.parent


def declared(header):
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b((?:fsv|fsvg)_[a-z0-9_]+)\s*\(", text)))


def test_fastsv_exports_every_declared_symbol():
    lib = _native.fastsv_lib()
    names = declared("fastsv.h")
    assert "fsv_upload_csr" in names and "fsv_run" in names and "fsv_nccl_attach" in names
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_native.FASTSV_SYMBOLS)


def test_graphgen_exports_every_declared_symbol():
    lib = _native.graphgen_lib()
    names = declared("fsv_graphgen.h")
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_native.GRAPHGEN_SYMBOLS)


def test_abi_version_and_error_string():
    lib = _native.fastsv_lib()
    assert lib.fsv_abi_version() == 5
    assert isinstance(_native.last_error(), str)


def test_null_context_is_a_contract_error():
    lib = _native.fastsv_lib()
    assert lib.fsv_destroy(None) == 0
    assert lib.fsv_set_stream(None, None) == 2
    assert lib.fsv_solve(None, None, None) == 2
    assert "NULL" in _native.last_error()


def test_no_cpu_fallback_without_device():
    if fb.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(fb.DeviceError):
        fb.Solver(0)
    with pytest.raises(fb.DeviceError):
        fb.fastsv_la(fb.build_csr(3, [(0, 1)]))
    with pytest.raises(fb.DeviceError):
        fb.require_device()
