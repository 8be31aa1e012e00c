"""Build recipes for the native pieces (in-tree, no JIT cache).

- ``libfastsv.so``   — the sm_100a CUDA kernels + C-ABI (include/fastsv.h),
                       nvcc ``-gencode arch=compute_100a,code=sm_100a``.
- ``libfsv_graphgen.so`` — host generators + CSR builder (include/fsv_graphgen.h).
- ``oracle/liborcale.so`` — the CPU parity checker (test infrastructure).

``python -m paper_1910_05971_b200.build`` builds everything.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
ORACLE = ROOT / "oracle"

LIB_FASTSV = PKG / "libfastsv.so"
LIB_GRAPHGEN = PKG / "libfsv_graphgen.so"
LIB_ORACLE = ORACLE / "liboracle.so"

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = shutil.which("nvcc") or os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CUDA_SOURCES = ["fastsv.cu"]
CUDA_HEADERS = ["fsv_kernels.cuh", "fsv_variants.cuh", "philox.h"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True)


def build_graphgen(force=False, verbose=False) -> Path:
    src = CSRC / "fsv_graphgen.cpp"
    deps = [src, CSRC / "philox.h", INCLUDE / "fsv_graphgen.h"]
    if force or _stale(LIB_GRAPHGEN, deps):
        _run(["g++", "-O3", "-march=x86-64-v3", "-std=c++17", "-fopenmp", "-fPIC", "-shared",
              "-I", INCLUDE, "-o", LIB_GRAPHGEN, src], verbose)
    return LIB_GRAPHGEN


def build_oracle(force=False, verbose=False) -> Path:
    src = ORACLE / "fsv_oracle.c"
    if force or _stale(LIB_ORACLE, [src]):
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", LIB_ORACLE, src], verbose)
    return LIB_ORACLE


def build_fastsv(force=False, verbose=False, extra_flags=()) -> Path:
    srcs = [CSRC / s for s in CUDA_SOURCES]
    deps = srcs + [CSRC / h for h in CUDA_HEADERS] + [INCLUDE / "fastsv.h"]
    if force or _stale(LIB_FASTSV, deps):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
               "-cudart", "static", "-Xcompiler", "-fopenmp", "-I", INCLUDE, "-Xptxas", "-v" if verbose else "-O3",
               *extra_flags, "-o", LIB_FASTSV, *srcs, "-ldl", "-lpthread", "-lgomp"]
        _run(cmd, verbose)
    return LIB_FASTSV


LIB_FASTSV_CHECKED = PKG / "libfastsv_checked.so"


def build_fastsv_checked(force=False, verbose=False) -> Path:
    """Bounds-checked build (-DFSV_CHECKS) for the tests: every vertex-array
    load and min-reduction of a solve must hit a registered buffer, else the
    kernel traps. Not used by the product path."""
    srcs = [CSRC / s for s in CUDA_SOURCES]
    deps = srcs + [CSRC / h for h in CUDA_HEADERS] + [INCLUDE / "fastsv.h"]
    if force or _stale(LIB_FASTSV_CHECKED, deps):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
               "-cudart", "static", "-Xcompiler", "-fopenmp", "-I", INCLUDE, "-DFSV_CHECKS", "-o", LIB_FASTSV_CHECKED, *srcs,
               "-ldl", "-lpthread", "-lgomp"]
        _run(cmd, verbose)
    return LIB_FASTSV_CHECKED


def build_all(force=False, verbose=False):
    return [build_graphgen(force, verbose), build_oracle(force, verbose),
            build_fastsv(force, verbose), build_fastsv_checked(force, verbose)]


if __name__ == "__main__":
    force = "--force" in sys.argv
    for p in build_all(force=force, verbose=True):
        print("built", p)
