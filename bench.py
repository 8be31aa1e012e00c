"""Benchmark: edges/sec to convergence of B200 FastSV (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

A step = one full FastSV solve (iteration 1 .. convergence) of the config's
graph, the device layout resident in HBM when the timed region starts.
`value` = |E| / mean step time (|E| = undirected input edges as generated).
Beside it: `layout` (device-resident CSR -> oriented layout, and the one-shot
CSR-resident -> labels throughput), `e2e` (pinned host CSR -> fsv_upload_csr
-> solve -> labels D2H through the C ABI) and `api` (the public drop-in
fastsv_la(g) on pageable numpy arrays, wall clock, RunResult with Labeling).

N > 1: one rank per GPU (torchrun; `--gpus N` without torchrun re-launches
itself under torch.distributed.run), 1D row partition balanced by entries,
per-iteration NCCL allreduce-min of the next-parent vector inside the
library; step time is the max over ranks.

--impl reference: the UNMODIFIED reference `svcc` (installed into
baseline/_ref) runs svcc.fastsv_la(g, DriverConfig(workers=cores)) on the
host cores, rank 0 only, on the same graph regenerated in pure numpy
(baseline/ref_inputs.py) so no library of this repo is mapped into it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured"
        except Exception:
            pass
    return PEAKS_FALLBACK["hbm_gbs"], "fallback"


class ClockSampler:
    """SM clock + throttle-reason sampling DURING the timed region (NVML polled
    every ~2 ms from a thread; falls back to nothing if NVML is unavailable)."""

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = self.dev
            if vis:
                try:
                    idx = int(vis.split(",")[self.dev])
                except ValueError:
                    idx = self.dev
            self._h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self._nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
            return
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        if self._t is None:
            return None
        self._stop.set()
        self._t.join(timeout=2)
        nv = self._nv
        names = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
                 "hw_power_brake": nv.nvmlClocksEventReasonHwPowerBrakeSlowdown}
        if not self.samples:
            return None
        reasons = sorted({k for _, r in self.samples for k, bit in names.items() if r & bit})
        sm = [a for a, _ in self.samples]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "source": "nvml"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_graph(config: int, scale: int | None):
    from paper_1910_05971_b200 import build_csr
    from paper_1910_05971_b200 import generators as gen
    n, pairs = gen.baseline_graph(config, scale)
    g = build_csr(n, pairs)
    return n, pairs, g


def row_partition(offsets: np.ndarray, world: int, rank: int):
    """Contiguous row range whose entry count is ~m/world."""
    n = offsets.size - 1
    m = int(offsets[-1])
    lo = int(np.searchsorted(offsets, m * rank // world, side="left")) if rank else 0
    hi = int(np.searchsorted(offsets, m * (rank + 1) // world, side="left")) if rank + 1 < world else n
    return min(lo, n), min(hi, n)


def bytes_model(g):
    n, m = g.n, g.m
    s_off = 4 if m < 2 ** 31 else 8
    hook = 4 * m + s_off * (n + 1) + 12 * n  # adjacency + offsets + read f, read gf, write f'
    it = 4 * m + s_off * (n + 1) + 24 * n    # SURVEY §8(d) B_iter
    return hook, it


def _import_svcc():
    """The reference package from baseline/_ref (pip --target install), or None."""
    ref = ROOT / "baseline" / "_ref"
    if (ref / "svcc").is_dir() and str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import svcc  # noqa: F401
        return svcc
    except ImportError:
        return None


def run_reference(args, world, rank):
    """CPU reference arm: the unmodified svcc.fastsv_la on all host cores."""
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    from baseline import ref_inputs
    t0 = time.perf_counter()
    if args.scale is not None and args.config in (2, 5):
        n, pairs = ref_inputs.rmat(args.scale, 16, seed=0)
    else:
        n, pairs = ref_inputs.baseline_graph(args.config)
    off, cols = ref_inputs.csr(n, pairs)
    prep_s = time.perf_counter() - t0
    edges = int(pairs.shape[0])
    del pairs
    svcc = _import_svcc()
    if svcc is not None:
        off.flags.writeable = False
        cols.flags.writeable = False
        g = svcc.CsrGraph(n=n, row_offsets=off, col_indices=cols)
        cfg = svcc.DriverConfig(workers=cores)

        def step():
            r = svcc.fastsv_la(g, cfg)
            return r.iterations
        kind, what = "reference", f"svcc.fastsv_la(g, DriverConfig(workers={cores})) from baseline/_ref"
    else:
        from oracle import port   # numpy restatement, used only when svcc is not installed
        pg = port.PortGraph(n, off, cols)

        def step():
            return port.fastsv_la(pg, workers=cores)[1]
        kind, what = "port", f"numpy port of svcc.fastsv_la (oracle/port.py), workers={cores}"
    for _ in range(args.warmup):
        iters = step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        iters = step()
        times.append(time.perf_counter() - t0)
    step_s = sum(times) / len(times)
    val = edges / step_s
    extra = {}
    if svcc is not None and not args.no_cpu_baseline:
        # the vertex-level twin, single-threaded
        t0 = time.perf_counter()
        r = svcc.fastsv(g)
        extra = {"svcc.fastsv_1thread_s": time.perf_counter() - t0, "svcc.fastsv_iterations": r.iterations}
    line = {
        "metric": "edges/sec to convergence (|E|/time)", "value": val, "unit": "edges/s",
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded generator, BASELINE config)",
        "config": {"workload": f"config{args.config} (BASELINE.json configs[{args.config - 1}])",
                   "n": n, "edges": edges, "m_dir": int(off[-1]), "iterations": iters,
                   "parallelism": "host threads (reference CPU path)"},
        "cpu_baseline": {"value": val, "unit": "edges/s", "cores": cores, "kind": kind,
                         "sample": f"full solve of config {args.config} per step: {what}"},
        "e2e": {"value": val, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "input_prep_s": prep_s,
        **extra,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(g, n_edges, budget_s=20.0):
    """Bounded timing of the reference itself (svcc.fastsv_la from
    baseline/_ref, all host cores) on this host; the numpy port stands in
    only when the reference is not installed."""
    cores = len(os.sched_getaffinity(0))
    svcc = _import_svcc()
    if svcc is not None:
        off = np.ascontiguousarray(g.row_offsets, dtype=np.int64)
        cols = np.ascontiguousarray(g.col_indices, dtype=np.int64)
        rg = svcc.CsrGraph(n=g.n, row_offsets=off, col_indices=cols)
        cfg = svcc.DriverConfig(workers=cores)
        run = lambda: svcc.fastsv_la(rg, cfg)  # noqa: E731
        kind, what = "reference", f"svcc.fastsv_la from baseline/_ref, workers={cores}"
    else:
        from oracle import port
        pg = port.PortGraph(g.n, g.row_offsets, g.col_indices)
        run = lambda: port.fastsv_la(pg, workers=cores)  # noqa: E731
        kind, what = "port", f"numpy port of svcc.fastsv_la, workers={cores}"
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s / 2 or len(times) >= 3:
            break
    best = min(times)
    return {"value": n_edges / best, "unit": "edges/s", "cores": cores, "kind": kind,
            "sample": f"{len(times)} full solve(s) of the same graph, best taken ({best:.2f} s each; {what})"}


def spawn_ranks(args) -> int:
    """`--gpus N` without torchrun: re-launch under torch.distributed.run with
    one rank per GPU; refuse (non-zero exit) when fewer GPUs are visible."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}", file=sys.stderr)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, help="BASELINE.json config number (1-5)")
    ap.add_argument("--scale", type=int, default=None, help="override generator scale (dev only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--hub-slots", type=int, default=0)
    ap.add_argument("--tile", type=int, default=0,
                    help="column-range tiling of the layout (vertices per tile, -1 auto, 0 off)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_env()

    if args.impl == "reference":
        # CPU arm: rank 0 works, the other ranks exit without work
        run_reference(args, max(world, args.gpus) if "WORLD_SIZE" not in os.environ else world, rank)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)

    import torch
    import torch.distributed as dist
    import paper_1910_05971_b200 as fb

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    n, pairs, g = make_graph(args.config, args.scale)
    n_edges = int(pairs.shape[0])
    del pairs
    solver = fb.Solver(local, hub_slots=args.hub_slots)
    if args.tile:
        solver.set_tile_width(args.tile)
    # one dedicated (non-default) stream for the solver, the L2 flush and the
    # timing events: the legacy default stream is not ordered against the
    # library's non-blocking stream, so flush/events/solve must share this one
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    solver.set_stream(stream.cuda_stream)
    if world > 1:
        uid = [fb.Solver.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        solver.attach_nccl(uid[0], world, rank)
    lo, hi = row_partition(g.row_offsets, world, rank) if world > 1 else (0, n)
    offsets = np.ascontiguousarray(g.row_offsets)
    cols_slice = np.ascontiguousarray(g.col_indices[offsets[lo]:offsets[hi]])
    solver.upload(g, lo, hi, cols_slice)

    # L2 flush between steps (outside the timed events): write a buffer
    # larger than the 126 MB L2, then read a second one, so the flush's own
    # dirty lines are written back before the timed region instead of during
    # it (the solve starts with none of its data in L2 either way)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush_rd = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
    flush_sink = torch.empty(1, dtype=torch.int64, device="cuda")

    def flush_l2():
        flush.zero_()
        torch.sum(flush_rd.view(torch.int64), dim=0, keepdim=True, out=flush_sink)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        solver.solve()
    labels = solver.labels()
    st = solver.stats
    iters = int(st.iterations)

    # ---- timed region: K device-resident solves -------------------------
    sampler = ClockSampler(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches = 0
    barrier()
    sampler.start()
    for i in range(args.steps):
        flush_l2()                         # evict L2 (not timed)
        ev[i][0].record(stream)
        s = solver.solve()
        ev[i][1].record(stream)
        launches += int(s.kernel_launches)
    barrier()
    clocks = sampler.stop()
    step_ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    t = torch.tensor([step_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms = float(t.item())

    # ---- per-kernel profile pass (events around every kernel) -----------
    prof = []
    for _ in range(3):
        flush_l2()
        prof.append(fb.FsvStats.from_buffer_copy(solver.solve(profile=True)))   # solve() reuses one struct
    best = min(prof, key=lambda p: p.solve_ms)
    hook_ms = best.hook_ms                 # dense k_hook launches only
    hook_launches = best.hook_launches
    solve_ms_prof = best.solve_ms
    kernel_ms = {"k_first": best.first_ms, "k_hook(dense)": best.hook_ms,
                 "k_hook(sparse push)": best.push_ms, "k_hubfix": best.hubfix_ms,
                 "k_shortcut": best.shortcut_ms, "allreduce": best.allreduce_ms}

    # ---- e2e: host CSR -> upload -> solve -> labels (public C-ABI path) ----
    pin_off = torch.from_numpy(offsets.copy()).pin_memory()
    pin_cols = torch.from_numpy(cols_slice.copy()).pin_memory()
    pin_lab = torch.empty(n, dtype=torch.int32).pin_memory()
    e2e_times = []
    for i in range(max(2, min(args.steps, 5))):
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        solver.upload_arrays(n, pin_off.data_ptr(), pin_cols.data_ptr(), lo, hi)
        solver.solve()
        solver.labels_into(pin_lab.data_ptr())
        b.record(stream)
        torch.cuda.synchronize()
        e2e_times.append(a.elapsed_time(b))
    e2e_ms = sum(e2e_times[1:]) / max(1, len(e2e_times) - 1)
    # the copy-engine floor of the same host buffers, for the breakdown
    d_off = torch.empty_like(pin_off, device="cuda")
    d_cols = torch.empty_like(pin_cols, device="cuda")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    d_off.copy_(pin_off, non_blocking=True)
    d_cols.copy_(pin_cols, non_blocking=True)
    b.record(stream)
    torch.cuda.synchronize()
    h2d_floor_ms = a.elapsed_time(b)
    del d_off, d_cols
    te = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    assert np.array_equal(pin_lab.numpy(), labels), "e2e labels differ from resident-solve labels"

    # ---- layout: device-resident CSR -> oriented layout (fsv_upload_csr_device)
    # The CSR (the reference's input structure, graph.py:20-52) sits in HBM;
    # the layout build reads it in place. One-shot throughput = |E| /
    # (layout + solve): what a single solve of a freshly resident graph costs.
    d_off_t = torch.from_numpy(offsets.copy()).to("cuda")
    d_cols_t = torch.from_numpy(cols_slice.copy()).to("cuda")
    lay_times, lay_solve = [], []
    for i in range(max(3, min(args.steps, 6))):
        barrier()
        flush_l2()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(stream)
        solver.upload_device(n, d_off_t.data_ptr(), d_cols_t.data_ptr(), lo, hi)
        b.record(stream)
        solver.solve()
        c.record(stream)
        torch.cuda.synchronize()
        if i:
            lay_times.append(a.elapsed_time(b))
            lay_solve.append(b.elapsed_time(c))
    layout_ms = sum(lay_times) / len(lay_times)
    oneshot_ms = layout_ms + sum(lay_solve) / len(lay_solve)
    tl = torch.tensor([layout_ms, oneshot_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tl, op=dist.ReduceOp.MAX)
    layout_ms, oneshot_ms = (float(x) for x in tl.tolist())
    assert np.array_equal(solver.labels(), labels), "device-CSR upload labels differ"

    # ---- api: the public drop-in on pageable host arrays (wall clock) ----
    api = None
    if world == 1:
        fb.fastsv_la(g, device=local)   # context creation + first upload
        api_times = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = fb.fastsv_la(g, device=local)
            api_times.append((time.perf_counter() - t0) * 1e3)
        assert np.array_equal(r.labeling.labels, labels.astype(np.int64)), "api labels differ"
        api = {"ms_per_call": min(api_times), "value": n_edges / (min(api_times) * 1e-3), "unit": "edges/s",
               "call": "paper_1910_05971_b200.fastsv_la(g) -> RunResult (pageable numpy CsrGraph in, "
                       "Labeling with sizes out; upload + layout + solve + trace + device Labeling)",
               "components": r.labeling.component_count}

    if rank == 0:
        peak, peak_kind = load_peaks()
        hook_bytes, iter_bytes = bytes_model(g)
        if world > 1:
            hook_bytes = (4 * g.m + (4 if g.m < 2 ** 31 else 8) * (n + 1)) // world + 12 * n
        per_launch_ms = hook_ms / max(hook_launches, 1)
        achieved = hook_bytes / (per_launch_ms * 1e-3) / 1e9 if hook_launches else 0.0
        traffic = None
        tfile = ROOT / "profiles" / "hook_traffic.json"
        if tfile.exists():
            try:
                td = json.loads(tfile.read_text())
                if td.get("config") == args.config and td.get("n") == n:
                    traffic = td.get("bytes_per_launch")
            except Exception:
                traffic = None
        line = {
            "metric": "edges/sec to convergence (|E|/time)",
            "value": n_edges / (step_ms * 1e-3),
            "unit": "edges/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "int32",
            "data": "synthetic (seeded Philox/PCG64 generator of the BASELINE config)",
            "config": {"workload": f"config{args.config} (BASELINE.json configs[{args.config - 1}])",
                       "n": n, "edges": n_edges, "m_dir": g.m, "iterations": iters,
                       "oriented_entries": int(st.oriented_entries), "hub_slots": int(st.hub_slots),
                       "minority_sweep_iterations": int(st.minority_iterations),
                       "l2": "flushed between steps (256 MiB write + 256 MiB read, outside the timed events)",
                       "layout_tiles": args.tile,
                       "parallelism": f"edge-partition x{world}" if world > 1 else "single GPU"},
            "iteration_model": {"bytes_per_iter": iter_bytes,
                                "frac_of_hbm": iters * iter_bytes / (step_ms * 1e-3) / 1e9 / peak},
            "roofline": {"kernel": "k_hook", "bound": "hbm", "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "bytes_per_launch": hook_bytes,
                         "launch_ms": per_launch_ms, "launches": hook_launches,
                         "share_of_step": hook_ms / solve_ms_prof if solve_ms_prof else None,
                         "step_breakdown_ms": kernel_ms, "profiled_step_ms": solve_ms_prof,
                         "note": "launches = k_hook launches of dense iterations (mean duration); "
                                 f"{int(st.minority_iterations)} of them took the minority sweep, which visits only "
                                 "the edges at vertices outside the majority grandparent and moves far less "
                                 "than bytes_per_launch; per-launch split in DESIGN.md section 8"},
            "e2e": {"value": n_edges / (e2e_ms * 1e-3), "unit": "edges/s",
                    "ms_per_step": e2e_ms,
                    "h2d_copy_floor_ms": h2d_floor_ms,
                    "path": "pinned host CSR -> fsv_upload_csr (H2D + layout build) -> fsv_solve -> fsv_get_labels",
                    "h2d_bytes_per_step": int(offsets.nbytes + cols_slice.nbytes),
                    "d2h_bytes_per_step": int(4 * n)},
            "layout": {"ms": layout_ms,
                       "path": "device CSR (int64 offsets, int32 columns in HBM) -> fsv_upload_csr_device "
                               "(degree order, hub table, oriented layout) ",
                       "oneshot_ms": oneshot_ms,
                       "value_incl_layout": n_edges / (oneshot_ms * 1e-3)},
            "api": api,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if world > 1:
            # NVLink roofline of the per-iteration exchange (dense iterations:
            # allreduce-min, ring bus bytes 2(P-1)/P*4n per GPU, SURVEY §8d;
            # sparse iterations: the delta lists) against the measured peer
            # bandwidth; bytes are the library's own count of what it sent
            xs = best.dense_exchanges + best.delta_exchanges
            x_ms = best.allreduce_ms / xs if (best.allreduce_ms and xs) else None
            x_bytes = best.exchange_bytes / xs if xs else None
            line["nvlink"] = {"collective": "ncclAllReduce(int32, min) of the next-parent vector (dense iterations); "
                                            "ncclAllGather of (index, value) deltas (sparse iterations)",
                              "dense_exchanges": int(best.dense_exchanges),
                              "delta_exchanges": int(best.delta_exchanges),
                              "bytes_per_exchange_per_gpu": x_bytes, "exchange_ms": x_ms,
                              "dense_allreduce_bus_bytes": 2 * (world - 1) / world * 4 * n,
                              "achieved": (x_bytes / (x_ms * 1e-3) / 1e9) if x_ms else None,
                              "peak": 770.0, "unit": "GB/s",
                              "peak_kind": "measured peer copy per direction (B200_PROFILING.md)",
                              "frac": (x_bytes / (x_ms * 1e-3) / 1e9 / 770.0) if x_ms else None}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_sample(g, n_edges)
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
