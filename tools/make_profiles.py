"""Summarise ncu outputs into profiles/ (run here, after a gpurun brought them back).

    python tools/make_profiles.py --launches gpurun_out/launches_r01.csv \
        --full gpurun_out/hook_r01.ncu-rep --out profiles/r01 --config 2

Writes
  <out>/launches_summary.txt   per-kernel launch count, mean/total device time, share
  <out>/hook_full_summary.txt  key ncu --set full metrics of each captured k_hook launch
  profiles/hook_traffic.json   DRAM bytes per dense k_hook launch (bench.py `traffic`)
"""

from __future__ import annotations

import argparse
import csv
import json
import subprocess
from collections import OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

FULL_KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "lts__t_requests_srcunit_tex_op_red.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]


def launches(path: Path, out: Path):
    rows = list(csv.reader(path.read_text().splitlines()))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3,
              "msecond": v * 1e3}.get(unit, v / 1e3)
        name = r[ki].split("(")[0].replace("void ", "")
        agg.setdefault(name, []).append(us)
    solve = {"fsv::k_first", "fsv::k_hook", "fsv::k_hubfix", "fsv::k_shortcut", "fsv::k_solve_init",
             "k_f1_solve"}
    base = lambda k: k.split("<")[0]
    total = sum(sum(v) for v in agg.values())
    stotal = sum(sum(v) for k, v in agg.items() if base(k) in solve)
    lines = [f"source: {path.name} (ncu --metrics gpu__time_duration.sum --clock-control none;"
             " cold-cache, serialised launches: compare shares, not absolutes)",
             "share = of all launches (includes the e2e uploads' layout-build kernels);"
             " solve share = of the solve kernels only (the timed `value` region).",
             "ncu does not list kernels inside the solve's conditional CUDA-graph loop; the solve"
             " kernels below come from the bench's profiled (host-loop) pass of the same solve.",
             f"{'kernel':58s} {'n':>5s} {'mean us':>9s} {'total us':>10s} {'share':>7s} {'solve share':>11s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        ss = f"{sum(v)/stotal*100:10.1f}%" if base(k) in solve else ""
        lines.append(f"{k[:58]:58s} {len(v):5d} {sum(v)/len(v):9.1f} {sum(v):10.1f} {sum(v)/total*100:6.1f}% {ss}")
    (out / "launches_summary.txt").write_text("\n".join(lines) + "\n")
    print("\n".join(lines[:14]))


def full(path: Path, out: Path, config: int, n: int | None):
    txt = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]
    lines = [f"source: {path.name} (ncu --set full --clock-control none)"]
    traffic = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        lines.append(f"---- {name}")
        for k in FULL_KEYS:
            if k in h:
                lines.append(f"  {k:62s} {r[h.index(k)]}")
        st = [(float(r[i] or 0), c) for i, c in enumerate(h)
              if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("per_issue_active.ratio")]
        st.sort(reverse=True)
        lines.append("  stalls/issue: " + ", ".join(
            f"{c.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, c in st[:6]))
        if "k_hook" in name:
            rd = float(r[h.index("dram__bytes_read.sum")]) * 1e6
            wr = float(r[h.index("dram__bytes_write.sum")]) * 1e6
            inst = float(r[h.index("smsp__inst_executed.sum")])
            if inst > 8e6:          # launches of dense iterations: the sweep (> 9e7 instructions on
                traffic.append(rd + wr)   # config 2) and the minority sweep (1e7); the sparse push has 6e6
    (out / "hook_full_summary.txt").write_text("\n".join(lines) + "\n")
    if traffic:
        rec = {"config": config, "n": n, "bytes_per_launch": sum(traffic) / len(traffic),
               "launches_captured": len(traffic), "source": str(out / path.name)}
        (ROOT / "profiles" / "hook_traffic.json").write_text(json.dumps(rec, indent=1) + "\n")
        print("hook traffic per dense launch:", rec["bytes_per_launch"] / 1e6, "MB")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", type=Path)
    ap.add_argument("--full", type=Path)
    ap.add_argument("--out", type=Path, required=True)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=1 << 22)
    a = ap.parse_args()
    a.out.mkdir(parents=True, exist_ok=True)
    if a.launches:
        launches(a.launches, a.out)
    if a.full:
        full(a.full, a.out, a.config, a.n)


if __name__ == "__main__":
    main()
