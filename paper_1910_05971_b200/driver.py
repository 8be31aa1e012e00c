"""The drop-in solver entry points (mirror svcc.driver / svcc.algorithms).

``fastsv_la`` and ``fastsv`` keep the reference signatures
(/root/reference/pkg/src/svcc/driver.py:64-65, algorithms.py:152-153) and
result types (``RunResult``/``IterationTrace``, algorithms.py:38-57), but
every iteration runs on a B200 through the C ABI of include/fastsv.h:

    Solver.upload(g)  -> fsv_upload_csr   (device oriented layout)
    Solver.run()      -> fsv_run          (whole FastSV loop on device)

No Triton, no multi-backend dispatch, no CPU fallback: without the CUDA
library or a device these calls raise.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import FsvConfig, FsvStats
from .errors import DeviceError, InputError, raise_for_status
from .graph import ID_DTYPE, ComponentSizes, CsrGraph, Labeling

_FORCE_MODES = ("auto", "dense_only", "sparse_only")


@dataclass(frozen=True)
class DriverConfig:
    """Same fields and validation as svcc.DriverConfig (driver.py:31-48).

    ``sparse_threshold``/``force_kernel`` select the per-iteration product
    exactly as the reference does (dense pull over the oriented layout, or a
    sparse push from the vertices whose gf changed); results are identical
    either way (test_driver.py:60-71) and the trace's kernel/flops fields
    follow the reference's definitions. ``workers`` is accepted for
    signature parity (the device decides its own parallelism).
    ``batch`` is B200-only: iterations queued per host convergence check."""

    sparse_threshold: float = 0.1
    force_kernel: str = "auto"
    workers: int = 1
    batch: int = 0

    def __post_init__(self):
        if not 0.0 <= self.sparse_threshold <= 1.0:
            raise ValueError(f"sparse_threshold must be in [0, 1], got {self.sparse_threshold}")
        if self.force_kernel not in _FORCE_MODES:
            raise ValueError(f"force_kernel must be one of {_FORCE_MODES}")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.batch < 0:
            raise ValueError("batch must be >= 0")


def choose_kernel(gf_changed: int, n: int, cfg: DriverConfig) -> str:
    """The reference's product-selection rule, strict inequality
    (driver.py:51-61; test_driver.py:29-38)."""
    if cfg.force_kernel == "dense_only":
        return "dense"
    if cfg.force_kernel == "sparse_only":
        return "sparse"
    return "sparse" if gf_changed < cfg.sparse_threshold * n else "dense"


@dataclass(frozen=True)
class HookingConfig:
    """svcc.HookingConfig (algorithms.py:28-35). All flags (FastSV proper)
    runs on the optimised path; weaker flag sets (the sv1..sv4 ablation,
    SURVEY §8f-3) run on the generic variant kernels with the same results
    as the reference."""

    grandparent_hooking: bool = True
    stochastic_hooking: bool = True
    aggressive_hooking: bool = True
    early_termination: bool = True


@dataclass(frozen=True)
class IterationTrace:
    iteration: int
    gf_changed: int
    f_changed: int
    kernel: str
    elapsed: float
    flops: int = 0


@dataclass
class RunResult:
    labeling: Labeling
    iterations: int
    trace: list
    snapshots: list | None = field(default=None, repr=False)

    @property
    def total_elapsed(self) -> float:
        return sum(t.elapsed for t in self.trace)


def _check(code: int) -> None:
    if code:
        raise_for_status(code, _native.last_error())


class Solver:
    """One device context: owns the resident graph and the solve buffers.

    ``upload`` is the (untimed) layout build; ``solve`` is the hot path.
    Reusing a Solver across solves of the same graph keeps the layout
    resident, as the bench does."""

    def __init__(self, device: int = 0, hub_slots: int = 0):
        self._lib = _native.fastsv_lib()
        self._ctx = ctypes.c_void_p()
        _check(self._lib.fsv_create(int(device), ctypes.byref(self._ctx)))
        _check(self._lib.fsv_set_hub_slots(self._ctx, int(hub_slots)))
        self.device = device
        self.n = 0
        self.m = 0
        self.stats = FsvStats()

    # -- lifetime ---------------------------------------------------------
    def close(self):
        if self._ctx:
            self._lib.fsv_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- configuration ----------------------------------------------------
    def set_stream(self, stream_ptr: int) -> None:
        _check(self._lib.fsv_set_stream(self._ctx, ctypes.c_void_p(int(stream_ptr))))

    def set_hub_slots(self, slots: int) -> None:
        _check(self._lib.fsv_set_hub_slots(self._ctx, int(slots)))

    def set_minority_sweep(self, enable: bool) -> None:
        """Minority sweep of late dense iterations (fsv_set_minority_sweep;
        default on, results identical either way)."""
        _check(self._lib.fsv_set_minority_sweep(self._ctx, int(bool(enable))))

    def set_tile_width(self, vertices: int) -> None:
        """Column-range tiling of the next upload's layout (0 off, > 0 width,
        < 0 auto); pays off over repeated solves of hub-less graphs whose
        vectors overflow L2 (fsv_set_tile_width)."""
        _check(self._lib.fsv_set_tile_width(self._ctx, int(vertices)))

    def attach_nccl(self, unique_id: bytes, nranks: int, rank: int) -> None:
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        _check(self._lib.fsv_nccl_attach(self._ctx, buf, int(nranks), int(rank)))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(_native.fastsv_lib().fsv_nccl_unique_id(buf))
        return buf.raw

    # -- graph ------------------------------------------------------------
    def upload(self, g, row_begin: int = 0, row_end: int | None = None, cols=None) -> None:
        """Upload a CsrGraph (ours or the reference's). For a 1D partition pass
        the row range and the column slice of those rows."""
        n = int(g.n)
        offsets = np.ascontiguousarray(g.row_offsets, dtype=np.int64)
        if row_end is None:
            row_end = n
        if cols is None:
            cols = g.col_indices[offsets[row_begin]:offsets[row_end]] if n else g.col_indices
        cols = np.ascontiguousarray(cols)
        if cols.dtype == np.int32:
            fn = self._lib.fsv_upload_csr
        else:
            cols = cols.astype(np.int64, copy=False)
            fn = self._lib.fsv_upload_csr64
        _check(fn(self._ctx, n, offsets.ctypes.data, cols.ctypes.data if cols.size else None,
                  int(row_begin), int(row_end)))
        self.n = n
        self.m = int(offsets[-1]) if n else 0

    def upload_edges(self, n: int, edges, row_begin: int = 0, row_end: int | None = None) -> None:
        """Edge list in: the CsrGraph is built on the device with
        svcc.build_csr's semantics (graph.py:55-97: range check with the
        reference's message, self-loops dropped, both orientations,
        duplicates merged, rows sorted), then the layout (fsv_upload_edges)."""
        n = int(n)
        if n < 0:
            raise InputError(f"vertex count must be non-negative, got {n}")
        pairs = edge_pairs(edges)
        fn = self._lib.fsv_upload_edges if pairs.dtype == np.int32 else self._lib.fsv_upload_edges64
        row_end = n if row_end is None else int(row_end)
        _check(fn(self._ctx, n, int(pairs.shape[0]), pairs.ctypes.data if pairs.size else None,
                  int(row_begin), row_end))
        self.n = n
        cnt = ctypes.c_int64(0)
        _check(self._lib.fsv_get_csr(self._ctx, None, None, ctypes.byref(cnt)))
        self.m = int(cnt.value)

    def csr(self) -> CsrGraph:
        """The resident symmetric CSR (full row offsets, this context's
        columns) as a CsrGraph with the reference's int64 ids."""
        cnt = ctypes.c_int64(0)
        _check(self._lib.fsv_get_csr(self._ctx, None, None, ctypes.byref(cnt)))
        off = np.empty(self.n + 1, dtype=np.int64)
        cols = np.empty(int(cnt.value), dtype=np.int32)
        _check(self._lib.fsv_get_csr(self._ctx, off.ctypes.data, cols.ctypes.data if cols.size else None,
                                     ctypes.byref(cnt)))
        off.flags.writeable = False
        c64 = cols.astype(ID_DTYPE)
        c64.flags.writeable = False
        return CsrGraph(n=self.n, row_offsets=off, col_indices=c64)

    def upload_arrays(self, n: int, offsets_ptr: int, cols_ptr: int, row_begin: int = 0,
                      row_end: int | None = None, int64_cols: bool = False) -> None:
        """Upload from raw host pointers (e.g. pinned buffers) — the e2e path."""
        fn = self._lib.fsv_upload_csr64 if int64_cols else self._lib.fsv_upload_csr
        _check(fn(self._ctx, int(n), ctypes.c_void_p(offsets_ptr), ctypes.c_void_p(cols_ptr),
                  int(row_begin), int(n if row_end is None else row_end)))
        self.n = int(n)
        # CsrGraph.m: stored directed entries = row_offsets[n] (graph.py:34-37)
        self.m = int(ctypes.c_int64.from_address(int(offsets_ptr) + 8 * int(n)).value)

    def upload_device(self, n: int, offsets_ptr: int, cols_ptr: int, row_begin: int = 0,
                      row_end: int | None = None, m: int | None = None) -> None:
        """Build the layout from a CSR already in device memory (int64 offsets
        of the full graph, int32 columns of rows [row_begin, row_end)). The
        arrays are borrowed, not copied: keep them alive and unchanged until
        the next upload or close() (fsv_upload_csr_device)."""
        _check(self._lib.fsv_upload_csr_device(self._ctx, int(n), ctypes.c_void_p(int(offsets_ptr)),
                                               ctypes.c_void_p(int(cols_ptr)), int(row_begin),
                                               int(n if row_end is None else row_end)))
        self.n = int(n)
        if m is not None:
            self.m = int(m)

    # -- solve ------------------------------------------------------------
    @staticmethod
    def _config(batch: int = 0, max_iters: int = 0, profile: bool = False,
                policy: int = 0, threshold: float = 0.1, hooking: int = 0, exchange: int = 0) -> FsvConfig:
        cfg = FsvConfig()
        cfg.hooking = int(hooking)
        cfg.exchange = int(exchange)
        cfg.batch = int(batch)
        cfg.max_iters = int(max_iters)
        cfg.profile = int(bool(profile))
        cfg.sparse_policy = int(policy)
        cfg.sparse_threshold = float(threshold)
        return cfg

    def solve(self, batch: int = 0, max_iters: int = 0, profile: bool = False,
              policy: int = 0, threshold: float = 0.1, hooking: int = 0, exchange: int = 0) -> FsvStats:
        """Run to convergence; labels stay on the device. ``profile`` brackets
        every kernel with CUDA events (per-kernel *_ms in the stats).
        ``policy``: 0 reference default (auto, 0.1), 1 dense only, 2 sparse
        only, 3 auto with ``threshold`` (svcc.choose_kernel). ``hooking``: 0
        all-flags FastSV, else HOOKING_SET | flag bits (a HookingConfig
        variant; HOOKING_SET alone is simplified_sv). ``exchange`` (multi-rank
        only): 0 sparse iterations exchange delta lists, 1 allreduce always."""
        cfg = self._config(batch, max_iters, profile, policy, threshold, hooking, exchange)
        _check(self._lib.fsv_solve(self._ctx, ctypes.byref(cfg), ctypes.byref(self.stats)))
        return self.stats

    def labels(self, out: np.ndarray | None = None) -> np.ndarray:
        """Labels of the last solve: int32 (device id type) by default, int64
        (widened on the device) when ``out`` is an int64 array."""
        if out is None:
            out = np.empty(self.n, dtype=np.int32)
        if out.dtype == np.int32:
            _check(self._lib.fsv_get_labels(self._ctx, out.ctypes.data if out.size else None))
        else:
            cnt = ctypes.c_int64(0)
            _check(self._lib.fsv_get_labeling(self._ctx, out.ctypes.data if out.size else None, None, None, 0,
                                              ctypes.byref(cnt)))
        return out

    def labeling(self) -> Labeling:
        """The reference's Labeling (graph.py:100-125) of the last solve, built
        on the device: int64 labels, component count, and the sizes of the
        components (fsv_get_labeling); no host pass over n."""
        cnt = ctypes.c_int64(0)
        _check(self._lib.fsv_get_labeling(self._ctx, None, None, None, 0, ctypes.byref(cnt)))
        c = int(cnt.value)
        labels = np.empty(self.n, dtype=ID_DTYPE)
        reps = np.empty(c, dtype=ID_DTYPE)
        sizes = np.empty(c, dtype=ID_DTYPE)
        _check(self._lib.fsv_get_labeling(self._ctx, labels.ctypes.data if self.n else None,
                                          reps.ctypes.data if c else None, sizes.ctypes.data if c else None,
                                          c, ctypes.byref(cnt)))
        for a in (labels, reps, sizes):
            a.flags.writeable = False
        return Labeling(labels=labels, component_count=c, sizes=ComponentSizes(reps, sizes))

    def labels_into(self, ptr: int) -> None:
        _check(self._lib.fsv_get_labels(self._ctx, ctypes.c_void_p(ptr)))

    def trace(self, k: int | None = None, full: bool = False):
        """(gf_changed, f_changed, ms) — plus (kernel 0/1, flops) with full=True."""
        k = int(self.stats.iterations) if k is None else int(k)
        gfc = np.zeros(max(k, 1), dtype=np.int64)
        fc = np.zeros(max(k, 1), dtype=np.int64)
        ms = np.zeros(max(k, 1), dtype=np.float32)
        kern = np.zeros(max(k, 1), dtype=np.int32)
        flops = np.zeros(max(k, 1), dtype=np.int64)
        _check(self._lib.fsv_get_trace_ex(self._ctx, gfc.ctypes.data, fc.ctypes.data, ms.ctypes.data,
                                          kern.ctypes.data, flops.ctypes.data, k))
        if full:
            return gfc[:k], fc[:k], ms[:k], kern[:k], flops[:k]
        return gfc[:k], fc[:k], ms[:k]

    def run(self, batch: int = 0, max_iters: int = 0, snapshots: bool = False, snap_cap: int = 256,
            policy: int = 0, threshold: float = 0.1, full_trace: bool = False, hooking: int = 0,
            with_labels: bool = True):
        """Solve + copy out: (labels int32 or None, iterations, gf_changed,
        f_changed, per-iteration ms, snapshots or None[, kernel, flops])."""
        cfg = self._config(batch, max_iters, False, policy, threshold, hooking)
        n = self.n
        labels = np.empty(n if with_labels else 0, dtype=np.int32)
        iters = ctypes.c_int32(0)
        if snapshots:
            cap = int(snap_cap)
            snap = np.empty((cap, n), dtype=np.int32)
            gfc = np.zeros(cap, dtype=np.int64)
            fc = np.zeros(cap, dtype=np.int64)
            _check(self._lib.fsv_run_snapshots(self._ctx, ctypes.byref(cfg),
                                               labels.ctypes.data if n and with_labels else None,
                                               ctypes.byref(iters),
                                               gfc.ctypes.data, fc.ctypes.data,
                                               snap.ctypes.data if n else ctypes.c_void_p(1), cap))
            _check(self._lib.fsv_get_stats(self._ctx, ctypes.byref(self.stats)))
        else:
            _check(self._lib.fsv_solve(self._ctx, ctypes.byref(cfg), ctypes.byref(self.stats)))
            iters.value = self.stats.iterations
            if n and with_labels:
                self.labels(labels)
            snap = None
        k = int(iters.value)
        gfc2, fc2, ms, kern, flops = self.trace(k, full=True)
        out = (labels if with_labels else None, k, gfc2, fc2, ms, (snap[:k] if snap is not None else None))
        return out + (kern, flops) if full_trace else out


def group_run(solvers, snapshots: bool = False, snap_cap: int = 256, policy: int = 0,
              threshold: float = 0.1, batch: int = 0, exchange: int = 0):
    """Emulated rank group on one device (fsv_group_solve): each Solver holds
    one row range of the same graph (``upload(g, lo, hi, cols)``); the group
    is solved in lockstep with a device min-merge in place of the NCCL
    allreduce, running the rank-partitioned kernels. Returns rank 0's
    (labels, iterations, gf_changed, f_changed, snapshots or None, kernel,
    flops) and every rank's labels."""
    lib = _native.fastsv_lib()
    arr = (ctypes.c_void_p * len(solvers))(*[s._ctx.value for s in solvers])
    cfg = Solver._config(batch, 0, False, policy, threshold, 0, exchange)
    s0 = solvers[0]
    n = s0.n
    if snapshots:
        cap = int(snap_cap)
        snap = np.empty((cap, n), dtype=np.int32)
        gfc = np.zeros(cap, dtype=np.int64)
        fc = np.zeros(cap, dtype=np.int64)
        labels = np.empty(n, dtype=np.int32)
        iters = ctypes.c_int32(0)
        _check(lib.fsv_group_run_snapshots(arr, len(solvers), ctypes.byref(cfg),
                                           labels.ctypes.data if n else None, ctypes.byref(iters),
                                           gfc.ctypes.data, fc.ctypes.data,
                                           snap.ctypes.data if n else ctypes.c_void_p(1), cap))
        k = int(iters.value)
        snap = snap[:k]
        _check(lib.fsv_get_stats(s0._ctx, ctypes.byref(s0.stats)))
    else:
        _check(lib.fsv_group_solve(arr, len(solvers), ctypes.byref(cfg), ctypes.byref(s0.stats)))
        k = int(s0.stats.iterations)
        snap = None
    gfc, fc, _, kern, flops = s0.trace(k, full=True)
    all_labels = [s.labels() for s in solvers]
    return all_labels[0], k, gfc, fc, snap, kern, flops, all_labels


_solvers: dict = {}


def default_solver(device: int = 0) -> Solver:
    """Process-wide solver per device (context creation costs milliseconds)."""
    s = _solvers.get(device)
    if s is None:
        s = _solvers[device] = Solver(device)
    return s


TRACE_CAP = 4096   # iteration cap of the device trace (kTraceCap in csrc/fastsv.cu)
_POLICY = {"auto": 3, "dense_only": 1, "sparse_only": 2}
_KIND = {0: "dense", 1: "sparse", 2: "none"}

# fsv_config.hooking (include/fastsv.h)
HOOKING_SET = 0x100
HOOK_GRANDPARENT, HOOK_STOCHASTIC, HOOK_AGGRESSIVE, HOOK_EARLY_TERMINATION = 1, 2, 4, 8


def hooking_code(cfg: "HookingConfig") -> int:
    """fsv_config.hooking for a HookingConfig variant (algorithms.py:28-35)."""
    return (HOOKING_SET | (HOOK_GRANDPARENT if cfg.grandparent_hooking else 0)
            | (HOOK_STOCHASTIC if cfg.stochastic_hooking else 0)
            | (HOOK_AGGRESSIVE if cfg.aggressive_hooking else 0)
            | (HOOK_EARLY_TERMINATION if cfg.early_termination else 0))


def _result(labeling, iters, gfc, fc, ms, snaps, kern, flops) -> RunResult:
    trace = [IterationTrace(iteration=i + 1, gf_changed=int(gfc[i]), f_changed=int(fc[i]),
                            kernel=_KIND.get(int(kern[i]), "dense"),
                            elapsed=float(ms[i]) / 1e3, flops=int(flops[i]))
             for i in range(iters)]
    snapshots = None
    if snaps is not None:
        snapshots = []
        for s in snaps:
            a = s.astype(ID_DTYPE)
            a.flags.writeable = False
            snapshots.append(a)
    return RunResult(labeling=labeling, iterations=int(iters), trace=trace, snapshots=snapshots)


def _solve_graph(g, record_snapshots: bool, batch: int, device: int, policy: int = 0,
                 threshold: float = 0.1, hooking: int = 0) -> RunResult:
    solver = default_solver(device)
    solver.upload(g)
    # the reference records snapshots without a limit (driver.py:109-112):
    # start from a bound that covers FastSV's O(log n) iterations and grow it
    # for slow-converging variants (sv1..sv4) until the trace cap
    cap = max(64, 4 * int(np.log2(max(g.n, 2))) + 16)
    while True:
        try:
            _, iters, gfc, fc, ms, snaps, kern, flops = solver.run(
                batch=batch, snapshots=record_snapshots, snap_cap=cap, policy=policy,
                threshold=threshold, full_trace=True, hooking=hooking, with_labels=False)
            break
        except ValueError as e:
            if not record_snapshots or "iterations ran" not in str(e) or cap >= TRACE_CAP:
                raise
            cap = min(4 * cap, TRACE_CAP)
    # Labeling (labels, count, sizes) built on the device; the star check ran
    # in the final vertex pass (graph.py:109-125)
    return _result(solver.labeling(), iters, gfc, fc, ms, snaps, kern, flops)


def fastsv_la(g, cfg: DriverConfig | None = None, record_snapshots: bool = False,
              device: int = 0) -> RunResult:
    """FastSV in the matrix formulation (driver.py:64-120) on a B200.

    Per-iteration parent vectors, iteration count, gf_changed/f_changed and
    labels are bit-identical to the reference for every DriverConfig."""
    cfg = cfg or DriverConfig()
    # svcc.DriverConfig works too (it has no B200 `batch` field)
    return _solve_graph(g, record_snapshots, getattr(cfg, "batch", 0), device, _POLICY[cfg.force_kernel],
                        cfg.sparse_threshold)


def fastsv(g, cfg: HookingConfig | None = None, record_snapshots: bool = False,
           device: int = 0) -> RunResult:
    """All-flags FastSV (algorithms.py:152-167) on a B200; identical results
    to fastsv_la (the reference proves this, test_acceptance.py:207-218)."""
    cfg = cfg or HookingConfig()
    if hooking_code(cfg) != HOOKING_SET | 15:
        # weaker variants (the sv1..sv4 ablation) run on the generic variant
        # kernels (csrc/fsv_variants.cuh), same results as algorithms.py:79-114
        return _solve_graph(g, record_snapshots, 0, device, hooking=hooking_code(cfg))
    res = _solve_graph(g, record_snapshots, 0, device)
    for i, t in enumerate(res.trace):
        res.trace[i] = IterationTrace(t.iteration, t.gf_changed, t.f_changed, "none", t.elapsed, 0)
    return res


def simplified_sv(g, record_snapshots: bool = False, device: int = 0) -> RunResult:
    """Baseline SV (algorithms.py:66-76,145-149): guarded tree hooking onto
    parents plus shortcutting, two commits per iteration, until f is stable."""
    return _solve_graph(g, record_snapshots, 0, device, hooking=HOOKING_SET)


def sv_level_config(level: int) -> "HookingConfig":
    """Cumulative ablation configurations sv1..sv5 (algorithms.py:170-181)."""
    if level not in (1, 2, 3, 4, 5):
        raise ValueError(f"sv level must be 1..5, got {level}")
    return HookingConfig(grandparent_hooking=level >= 2, stochastic_hooking=level >= 3,
                         aggressive_hooking=level >= 4, early_termination=level >= 5)


def ablation_results(g, device: int = 0):
    """sv1 (simplified_sv) and sv2..sv5 (fastsv under sv_level_config), all
    on the device; insists the five labelings agree (algorithms.py:184-199)."""
    from .errors import InvariantError
    runs = [("sv1", simplified_sv(g, device=device))]
    for level in (2, 3, 4, 5):
        runs.append((f"sv{level}", fastsv(g, sv_level_config(level), device=device)))
    base = runs[0][1].labeling.labels
    for name, result in runs[1:]:
        if not np.array_equal(result.labeling.labels, base):
            raise InvariantError(f"ablation configuration {name} disagrees with sv1 labels")
    return runs


def ablation_suite(g, device: int = 0):
    """(config_name, iterations) for sv1..sv5 (algorithms.py:202-204)."""
    return [(name, result.iterations) for name, result in ablation_results(g, device)]


def edge_pairs(edges) -> np.ndarray:
    """(k, 2) contiguous int32/int64 array of an edge list, with build_csr's
    input rules (graph.py:63-69): any iterable of pairs or an integer array."""
    if isinstance(edges, np.ndarray) and edges.dtype in (np.int32, np.int64):
        pairs = edges
    else:
        pairs = np.asarray(list(edges) if not isinstance(edges, np.ndarray) else edges, dtype=ID_DTYPE)
    if pairs.size == 0:
        pairs = pairs.reshape(0, 2)
    if pairs.ndim != 2 or pairs.shape[1] != 2:
        raise InputError("edges must be (u, v) pairs")
    return np.ascontiguousarray(pairs)


def connected_components(n: int, edges, device: int = 0) -> np.ndarray:
    """Edge list in, label vector out (int64, minimum id per component).
    The CSR is built on the device (fsv_upload_edges), then FastSV runs."""
    n = int(n)
    solver = default_solver(device)
    solver.upload_edges(n, edges)
    if n == 0:
        return np.zeros(0, dtype=ID_DTYPE)
    solver.solve()
    return solver.labels(np.empty(n, dtype=ID_DTYPE))


def device_count() -> int:
    c = ctypes.c_int(0)
    code = _native.fastsv_lib().fsv_device_count(ctypes.byref(c))
    if code:
        return 0
    return int(c.value)


def require_device() -> None:
    if device_count() < 1:
        raise DeviceError("no CUDA device available; the B200 solver has no CPU fallback")


__all__ = ["DriverConfig", "HookingConfig", "IterationTrace", "RunResult", "Solver", "choose_kernel",
           "fastsv_la", "fastsv", "connected_components", "default_solver", "device_count",
           "require_device", "CsrGraph"]
