"""ctypes bindings of the two native libraries (the maintainer-side binding of
include/fastsv.h and include/fsv_graphgen.h).

There is no CPU fallback: if ``libfastsv.so`` is missing or no CUDA device is
present, the solver entry points raise. Build with
``python -m paper_1910_05971_b200.build`` (``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_uint64, c_void_p
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# FSV_LIB: dev override (a kernel-shape variant built by tools/variants.sh)
LIB_FASTSV_PATH = Path(os.environ["FSV_LIB"]).resolve() if os.environ.get("FSV_LIB") else _PKG / "libfastsv.so"
LIB_GRAPHGEN_PATH = _PKG / "libfsv_graphgen.so"

FSV_OK, FSV_ERR_INPUT, FSV_ERR_CONTRACT, FSV_ERR_INVARIANT, FSV_ERR_RUNTIME = 0, 1, 2, 3, 4


class FsvConfig(ctypes.Structure):
    _fields_ = [("max_iters", c_int32), ("batch", c_int32), ("profile", c_int32),
                ("sparse_policy", c_int32), ("sparse_threshold", c_double), ("hooking", c_int32),
                ("exchange", c_int32)]


class FsvStats(ctypes.Structure):
    _fields_ = [("iterations", c_int32), ("component_count", c_int32), ("n", c_int64),
                ("m_dir", c_int64), ("oriented_entries", c_int64), ("hub_slots", c_int32),
                ("host_syncs", c_int32), ("kernel_launches", c_int32), ("solve_ms", c_float),
                ("hook_ms", c_float), ("hubfix_ms", c_float), ("shortcut_ms", c_float),
                ("first_ms", c_float), ("allreduce_ms", c_float), ("push_ms", c_float),
                ("hook_launches", c_int32), ("sparse_iterations", c_int32),
                ("dense_exchanges", c_int32), ("delta_exchanges", c_int32), ("exchange_bytes", c_int64),
                ("minority_iterations", c_int32), ("reserved", c_int32)]


# symbol -> (restype, argtypes); mirrors include/fastsv.h one to one
FASTSV_SYMBOLS = {
    "fsv_last_error": (c_char_p, []),
    "fsv_abi_version": (c_int, []),
    "fsv_device_count": (c_int, [POINTER(c_int)]),
    "fsv_create": (c_int, [c_int, POINTER(c_void_p)]),
    "fsv_destroy": (c_int, [c_void_p]),
    "fsv_set_hub_slots": (c_int, [c_void_p, c_int]),
    "fsv_set_tile_width": (c_int, [c_void_p, c_int64]),
    "fsv_set_minority_sweep": (c_int, [c_void_p, c_int]),
    "fsv_set_stream": (c_int, [c_void_p, c_void_p]),
    "fsv_upload_csr": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int64]),
    "fsv_upload_csr64": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int64]),
    "fsv_upload_csr_device": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int64]),
    "fsv_upload_edges": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_int64]),
    "fsv_upload_edges64": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_int64]),
    "fsv_get_csr": (c_int, [c_void_p, c_void_p, c_void_p, POINTER(c_int64)]),
    "fsv_solve": (c_int, [c_void_p, POINTER(FsvConfig), POINTER(FsvStats)]),
    "fsv_get_stats": (c_int, [c_void_p, POINTER(FsvStats)]),
    "fsv_get_labels": (c_int, [c_void_p, c_void_p]),
    "fsv_get_labels64": (c_int, [c_void_p, c_void_p]),
    "fsv_get_labeling": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, POINTER(c_int64)]),
    "fsv_get_trace": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int32]),
    "fsv_get_trace_ex": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32]),
    "fsv_run": (c_int, [c_void_p, POINTER(FsvConfig), c_void_p, POINTER(c_int32), c_void_p,
                        c_void_p, c_int32]),
    "fsv_run_snapshots": (c_int, [c_void_p, POINTER(FsvConfig), c_void_p, POINTER(c_int32),
                                  c_void_p, c_void_p, c_void_p, c_int32]),
    "fsv_nccl_unique_id": (c_int, [c_void_p]),
    "fsv_nccl_attach": (c_int, [c_void_p, c_void_p, c_int, c_int]),
    "fsv_group_solve": (c_int, [c_void_p, c_int, POINTER(FsvConfig), POINTER(FsvStats)]),
    "fsv_group_run_snapshots": (c_int, [c_void_p, c_int, POINTER(FsvConfig), c_void_p, POINTER(c_int32),
                                        c_void_p, c_void_p, c_void_p, c_int32]),
}

GRAPHGEN_SYMBOLS = {
    "fsvg_set_threads": (None, [c_int]),
    "fsvg_get_threads": (c_int, []),
    "fsvg_permutation": (c_int, [c_int64, c_uint64, c_void_p]),
    "fsvg_rmat": (c_int64, [c_int, c_int64, c_double, c_double, c_double, c_uint64, c_int, c_void_p]),
    "fsvg_grid": (c_int64, [c_int64, c_int64, c_double, c_uint64, c_int, c_void_p]),
    "fsvg_forest": (c_int64, [c_int64, c_int, c_int, c_int, c_uint64, c_int, c_void_p,
                              POINTER(c_int64)]),
    "fsvg_csr_build": (c_int64, [c_int64, c_int64, c_void_p, c_void_p, c_void_p, POINTER(c_int64)]),
    "fsvg_csr_build64": (c_int64, [c_int64, c_int64, c_void_p, c_void_p, c_void_p, POINTER(c_int64)]),
    "fsvg_fnv1a64": (c_uint64, [c_void_p, c_int64]),
}

_libs: dict = {}


def _bind(path: Path, symbols: dict):
    if not path.exists():
        raise ImportError(
            f"{path.name} is not built ({path}); run `python -m paper_1910_05971_b200.build` "
            "— there is no CPU fallback")
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in symbols.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def fastsv_lib():
    """The CUDA solver library (loaded once)."""
    if "fastsv" not in _libs:
        _libs["fastsv"] = _bind(LIB_FASTSV_PATH, FASTSV_SYMBOLS)
    return _libs["fastsv"]


def graphgen_lib():
    """The host generator / CSR builder library (loaded once)."""
    if "graphgen" not in _libs:
        _libs["graphgen"] = _bind(LIB_GRAPHGEN_PATH, GRAPHGEN_SYMBOLS)
    return _libs["graphgen"]


def last_error() -> str:
    msg = fastsv_lib().fsv_last_error()
    return msg.decode() if msg else ""
