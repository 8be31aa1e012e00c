"""bench.py's JSON-line contract (the driver parses it): the reference arm on
the CPU here, our arm on a B200. Small generator scales keep both quick."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def run_bench(*args):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--scale", "12", "--steps", "2", "--warmup", "3")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["warmup"] >= 3 and d["steps"] == 2
    assert d["metric"] == "edges/sec to convergence (|E|/time)" and d["value"] > 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    # the unmodified reference from baseline/_ref when it is installed there
    svcc_installed = (ROOT / "baseline" / "_ref" / "svcc").is_dir()
    assert d["cpu_baseline"]["kind"] == ("reference" if svcc_installed else "port")
    assert d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"].startswith("config2")


def test_reference_arm_maps_no_repo_library():
    """The reference process regenerates its input in numpy: none of this
    repo's shared objects may be mapped into it (checked from /proc/self/maps
    at exit)."""
    code = (
        "import runpy, sys, atexit\n"
        "def chk():\n"
        "    maps = open('/proc/self/maps').read()\n"
        f"    bad = [l for l in maps.splitlines() if '{ROOT}' in l and '.so' in l]\n"
        "    print('REPO_SO', len(bad), bad[:3])\n"
        "atexit.register(chk)\n"
        f"sys.argv = ['bench.py', '--impl', 'reference', '--scale', '11', '--steps', '1', '--warmup', '3']\n"
        f"runpy.run_path('{ROOT / 'bench.py'}', run_name='__main__')\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "REPO_SO 0 []" in r.stdout, r.stdout[-2000:]


def test_gpus_flag_refuses_without_enough_devices():
    """--gpus N (no torchrun) re-launches itself with N ranks, or fails loudly
    when fewer GPUs are visible (never silently runs one rank)."""
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("enough GPUs here: the spawn itself is exercised on multi-GPU boxes")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode != 0 and "needs 2 visible GPUs" in r.stderr


@pytest.mark.gpu
def test_our_arm_line():
    d = run_bench("--scale", "16", "--steps", "3", "--warmup", "3")
    assert (BASE_KEYS | {"roofline", "gpu_launches", "clocks", "iteration_model"}) <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0 and d["higher_is_better"] is True
    rf = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(rf)
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1.5
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    assert d["gpu_launches"] > 0
    assert set(d["cpu_baseline"]) >= {"value", "unit", "cores", "kind", "sample"}
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert d["layout"]["ms"] > 0 and d["layout"]["oneshot_ms"] > d["layout"]["ms"]
    assert d["api"]["ms_per_call"] > 0 and d["api"]["components"] > 0
