"""Command line front end with the reference CLI's contract (svcc/cli.py:95-291),
driving the B200 solver: ``run`` (one algorithm, JSON report), ``ablation``
(sv1..sv5 as CSV) and ``frontier`` (per-iteration trace as CSV). Report and
CSV schemas follow pkg/README.md:81-92 / cli.py:66-84,155-184; exit codes
0 ok, 1 input error, 2 verification failure, 3 invariant violation
(cli.py:1-5,271-287), and 4 when the device path cannot run (there is no
CPU fallback).

    python -m paper_1910_05971_b200 run --input g.mtx --algo fastsv-la --verify

Graph files: MatrixMarket coordinate (pattern/integer/real, general or
symmetric; 1-based) or whitespace edge lists (0-based pairs, '#' comments,
n = 1 + max id), as svcc.graphio reads them (graphio.py:17-109). The
``generate`` subcommand of the reference (its test-graph families) is not
part of this package.
"""

from __future__ import annotations

import argparse
import csv
import json
import sys

import numpy as np

from .driver import (DriverConfig, HookingConfig, ablation_results, fastsv, fastsv_la, simplified_sv,
                     sv_level_config)
from .errors import DeviceError, InputError, InvariantError, VerificationError
from .graph import CsrGraph, build_csr

KERNEL_CHOICES = {"auto": "auto", "dense-only": "dense_only", "sparse-only": "sparse_only"}
HOOK_FLAGS = ("hook-grandparent", "hook-stochastic", "hook-aggressive", "early-termination")


# ---- graph files --------------------------------------------------------------

def _content_lines(path):
    """(line number, stripped text) of every line of a text file."""
    try:
        with open(path, "r", encoding="utf-8") as fh:
            text = fh.read()
    except OSError as exc:
        raise InputError(f"cannot read {path}: {exc}")
    return list(enumerate((ln.strip() for ln in text.splitlines()), start=1))


def read_matrix_market(path) -> CsrGraph:
    lines = _content_lines(path)
    if not lines or not lines[0][1].lower().startswith("%%matrixmarket"):
        raise InputError(f"{path}: missing MatrixMarket header at line 1")
    head = lines[0][1].lower().split()
    if len(head) < 5 or head[1] != "matrix":
        raise InputError(f"{path}: malformed header at line 1")
    layout, field, symmetry = head[2], head[3], head[4]
    if layout == "array":
        raise InputError(f"{path}: array (dense) format is unsupported")
    if layout != "coordinate":
        raise InputError(f"{path}: unknown format '{layout}' at line 1")
    if field not in ("pattern", "integer", "real"):
        raise InputError(f"{path}: unsupported field '{field}' at line 1")
    if symmetry not in ("general", "symmetric"):
        raise InputError(f"{path}: unsupported qualifier '{symmetry}' at line 1")
    size = None
    declared = 0
    pairs = []
    for lineno, line in lines[1:]:
        if not line or line.startswith("%"):
            continue
        tok = line.split()
        if size is None:
            if len(tok) != 3:
                raise InputError(f"{path}: expected 'rows cols nnz' at line {lineno}")
            try:
                nrows, ncols, declared = int(tok[0]), int(tok[1]), int(tok[2])
            except ValueError:
                raise InputError(f"{path}: non-integer dimension at line {lineno}")
            if nrows != ncols:
                raise InputError(f"{path}: adjacency matrix must be square ({nrows}x{ncols} at line {lineno})")
            size = nrows
            continue
        if len(tok) not in (2, 3):
            raise InputError(f"{path}: malformed entry at line {lineno}")
        try:
            i, j = int(tok[0]), int(tok[1])
        except ValueError:
            raise InputError(f"{path}: non-integer index at line {lineno}")
        if not (1 <= i <= size and 1 <= j <= size):
            raise InputError(f"{path}: index out of bounds at line {lineno}")
        pairs.append((i - 1, j - 1))
    if size is None:
        raise InputError(f"{path}: missing dimension line")
    if len(pairs) != declared:
        raise InputError(f"{path}: header declares {declared} entries, found {len(pairs)}")
    return build_csr(size, np.array(pairs, dtype=np.int64).reshape(-1, 2))


def read_edge_list(path) -> CsrGraph:
    pairs = []
    top = -1
    for lineno, line in _content_lines(path):
        if not line or line.startswith("#"):
            continue
        tok = line.split()
        if len(tok) != 2:
            raise InputError(f"{path}: expected two ids at line {lineno}")
        try:
            u, v = int(tok[0]), int(tok[1])
        except ValueError:
            raise InputError(f"{path}: non-integer token at line {lineno}")
        if u < 0 or v < 0:
            raise InputError(f"{path}: negative id at line {lineno}")
        pairs.append((u, v))
        top = max(top, u, v)
    return build_csr(top + 1, np.array(pairs, dtype=np.int64).reshape(-1, 2))


def load_graph(path: str, fmt: str = "auto") -> CsrGraph:
    if fmt == "auto":
        lines = _content_lines(path)
        fmt = "mm" if lines and lines[0][1].lower().startswith("%%matrixmarket") else "el"
    return read_matrix_market(path) if fmt == "mm" else read_edge_list(path)


# ---- verification (independent of the solver) -------------------------------

def min_id_components(g: CsrGraph) -> np.ndarray:
    """Minimum vertex id of every vertex's component, from scipy's graph
    search (an independent check for --verify, cli.py:56-60)."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    if g.n == 0:
        return np.zeros(0, dtype=np.int64)
    a = csr_matrix((np.ones(g.m, dtype=np.int8), np.asarray(g.col_indices), np.asarray(g.row_offsets)),
                   shape=(g.n, g.n))
    _, comp = connected_components(a, directed=False)
    rep = np.full(comp.max() + 1, g.n, dtype=np.int64)
    np.minimum.at(rep, comp, np.arange(g.n, dtype=np.int64))
    return rep[comp]


def _verify(g, result) -> None:
    if not np.array_equal(result.labeling.labels, min_id_components(g)):
        raise VerificationError("labeling disagrees with the union-find oracle")


# ---- commands -----------------------------------------------------------------

def _driver_config(args, parser) -> DriverConfig:
    try:
        return DriverConfig(sparse_threshold=args.threshold, force_kernel=KERNEL_CHOICES[args.kernel],
                            workers=args.threads)
    except ValueError as exc:
        parser.error(str(exc))


def _report(g, source, algorithm, config, result, verified) -> dict:
    trace = [{"iteration": t.iteration, "gf_changed": t.gf_changed, "f_changed": t.f_changed,
              "kernel": t.kernel, "flops": t.flops, "elapsed": t.elapsed} for t in result.trace]
    return {"graph": {"n": g.n, "m": g.m, "source": source}, "algorithm": algorithm, "config": config,
            "component_count": result.labeling.component_count, "iterations": result.iterations,
            "trace": trace, "total_elapsed": result.total_elapsed, "verified": verified}


def _write(text: str, path) -> None:
    if path:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


def _write_csv(rows, path) -> None:
    if path:
        with open(path, "w", encoding="utf-8", newline="") as fh:
            csv.writer(fh).writerows(rows)
    else:
        csv.writer(sys.stdout).writerows(rows)


def cmd_run(args, parser) -> None:
    g = load_graph(args.input, args.format)
    overrides = [getattr(args, f.replace("-", "_")) for f in HOOK_FLAGS]
    hook_args_given = args.sv_level is not None or any(v is not None for v in overrides)
    if args.algo != "fastsv" and hook_args_given:
        parser.error("--sv-level and --hook-* flags apply to --algo fastsv")
    if args.algo == "sv":
        result, config = simplified_sv(g), {}
    elif args.algo == "fastsv":
        base = sv_level_config(args.sv_level) if args.sv_level else HookingConfig()
        names = ("grandparent_hooking", "stochastic_hooking", "aggressive_hooking", "early_termination")
        chosen = {k: (getattr(base, k) if v is None else bool(v)) for k, v in zip(names, overrides)}
        result, config = fastsv(g, HookingConfig(**chosen)), chosen
    else:
        dcfg = _driver_config(args, parser)
        result = fastsv_la(g, dcfg)
        config = {"sparse_threshold": dcfg.sparse_threshold, "force_kernel": dcfg.force_kernel,
                  "workers": dcfg.workers}
    verified = None
    if args.verify:
        _verify(g, result)
        verified = True
    if args.labels_out:
        with open(args.labels_out, "w", encoding="utf-8") as fh:
            fh.writelines(f"{u} {lab}\n" for u, lab in enumerate(result.labeling.labels.tolist()))
    rep = _report(g, args.input, args.algo, config, result, verified)
    _write(json.dumps(rep, indent=2, sort_keys=True) + "\n", args.output)


def cmd_ablation(args, parser) -> None:
    g = load_graph(args.input, args.format)
    runs = ablation_results(g)
    want = min_id_components(g)
    for name, result in runs:
        if not np.array_equal(result.labeling.labels, want):
            raise VerificationError(f"{name} labeling disagrees with the oracle")
    base = runs[0][1].iterations
    rows = [["name", "iterations", "total_elapsed", "reduction_vs_sv1"]]
    for name, result in runs:
        red = (base - result.iterations) / base if base else 0.0
        rows.append([name, result.iterations, f"{result.total_elapsed:.6f}", f"{red:.4f}"])
    _write_csv(rows, args.output)


def cmd_frontier(args, parser) -> None:
    g = load_graph(args.input, args.format)
    result = fastsv_la(g, _driver_config(args, parser))
    rows = [["iteration", "gf_changed", "gf_changed_frac", "kernel", "flops", "elapsed"]]
    for t in result.trace:
        frac = t.gf_changed / g.n if g.n else 0.0
        rows.append([t.iteration, t.gf_changed, f"{frac:.6f}", t.kernel, t.flops, f"{t.elapsed:.6f}"])
    _write_csv(rows, args.output)


# ---- parser -------------------------------------------------------------------

class _Parser(argparse.ArgumentParser):
    def error(self, message):          # usage mistakes are input errors (exit 1)
        raise InputError(message)


def _at_least_one(text: str) -> int:
    v = int(text)
    if v < 1:
        raise argparse.ArgumentTypeError("must be >= 1")
    return v


def build_parser() -> _Parser:
    p = _Parser(prog="paper_1910_05971_b200", description="FastSV connected components on a B200")
    sub = p.add_subparsers(dest="command", required=True)

    def graph_args(sp):
        sp.add_argument("--input", required=True, help="graph file (MatrixMarket or edge list)")
        sp.add_argument("--format", choices=("auto", "mm", "el"), default="auto")

    def driver_args(sp):
        sp.add_argument("--threshold", type=float, default=0.1, help="changed fraction for the sparse product")
        sp.add_argument("--kernel", choices=tuple(KERNEL_CHOICES), default="auto")
        sp.add_argument("--threads", type=_at_least_one, default=1, help="accepted for compatibility")

    run = sub.add_parser("run", help="run one algorithm, JSON report")
    graph_args(run)
    run.add_argument("--algo", choices=("sv", "fastsv", "fastsv-la"), default="fastsv")
    run.add_argument("--sv-level", type=int, choices=(1, 2, 3, 4, 5), default=None)
    for flag in HOOK_FLAGS:
        run.add_argument(f"--{flag}", action=argparse.BooleanOptionalAction, default=None)
    driver_args(run)
    run.add_argument("--verify", action="store_true", help="check labels against an independent search")
    run.add_argument("--labels-out", default=None, help="write 'vertex label' lines")
    run.add_argument("--output", "-o", default=None)
    run.set_defaults(func=cmd_run)

    abl = sub.add_parser("ablation", help="sv1..sv5 iterations as CSV")
    graph_args(abl)
    abl.add_argument("--output", "-o", default=None)
    abl.set_defaults(func=cmd_ablation)

    fr = sub.add_parser("frontier", help="per-iteration trace as CSV")
    graph_args(fr)
    driver_args(fr)
    fr.add_argument("--output", "-o", default=None)
    fr.set_defaults(func=cmd_frontier)
    return p


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
        args.func(args, parser)
    except InputError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except VerificationError as exc:
        print(f"verification failed: {exc}", file=sys.stderr)
        return 2
    except InvariantError as exc:
        print(f"invariant violated: {exc}", file=sys.stderr)
        return 3
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except DeviceError as exc:         # no CUDA device / CUDA failure: no CPU fallback
        print(f"device error: {exc}", file=sys.stderr)
        return 4
    return 0
