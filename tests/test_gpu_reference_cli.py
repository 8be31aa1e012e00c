"""the reference's own CLI (svcc.cli, installed unmodified in
baseline/_ref) driven against the B200 backend through the reference's own
swap mechanism — the solver names imported by svcc/cli.py:15-17, which the
reference's tests monkeypatch (pkg/tests/test_cli.py:165-173). Every
subcommand that reaches the hot path (run --algo fastsv-la/fastsv/sv with
--verify and --sv-level, frontier, ablation) must print the same report /
CSV / labels and exit with the same code as the unpatched reference, apart
from the wall-clock fields (elapsed, total_elapsed)."""

import csv
import json
import sys
from pathlib import Path

import pytest

import paper_1910_05971_b200 as fb

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


@pytest.fixture(scope="module")
def svcc_cli():
    if not (REF / "svcc").is_dir():
        pytest.skip("the reference is not installed in baseline/_ref")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import svcc.cli
    return svcc.cli


def _strip_timing(obj):
    if isinstance(obj, dict):
        return {k: _strip_timing(v) for k, v in obj.items() if k not in ("elapsed", "total_elapsed")}
    if isinstance(obj, list):
        return [_strip_timing(v) for v in obj]
    return obj


def _csv_without(path, drop):
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    idx = [i for i, h in enumerate(rows[0]) if h in drop]
    return [[c for i, c in enumerate(r) if i not in idx] for r in rows]


def _graphs(tmp_path, cli):
    files = {}
    mm = tmp_path / "tri.mtx"
    mm.write_text("%%MatrixMarket matrix coordinate pattern symmetric\n6 6 6\n2 1\n3 2\n3 1\n5 4\n6 5\n6 4\n")
    files["tri"] = str(mm)
    specs = {"path64": ["--family", "path", "--n", "64"],
             "star10": ["--family", "star", "--n", "10"],
             "gnp": ["--family", "gnp", "--n", "800", "--p", "0.004", "--seed", "3"],
             "mix": ["--family", "component_mix", "--blocks", "5", "--block-n", "120", "--block-p", "0.03",
                     "--seed", "7"],
             "grid": ["--family", "grid2d", "--rows", "12", "--cols", "17"]}
    for name, flags in specs.items():
        out = tmp_path / f"{name}.el"
        assert cli.main(["generate", "--output", str(out), *flags]) == 0
        files[name] = str(out)
    return files


def _swap_to_b200(monkeypatch, cli):
    monkeypatch.setattr(cli, "fastsv_la", fb.fastsv_la)
    monkeypatch.setattr(cli, "fastsv", fb.fastsv)
    monkeypatch.setattr(cli, "simplified_sv", fb.simplified_sv)
    monkeypatch.setattr(cli, "ablation_results", fb.ablation_results)


def test_reference_cli_run_reports_identical(svcc_cli, tmp_path, monkeypatch):
    cli = svcc_cli
    files = _graphs(tmp_path, cli)
    variants = [["--algo", "fastsv-la", "--verify"],
                ["--algo", "fastsv-la", "--kernel", "sparse-only"],
                ["--algo", "fastsv-la", "--kernel", "dense-only", "--threshold", "0.5"],
                ["--algo", "fastsv", "--verify"],
                ["--algo", "fastsv", "--sv-level", "3"],
                ["--algo", "fastsv", "--no-hook-stochastic"],
                ["--algo", "sv", "--verify"]]
    for name, path in files.items():
        for v in variants:
            outs = []
            for swapped in (False, True):
                with monkeypatch.context() as m:
                    if swapped:
                        _swap_to_b200(m, cli)
                    rep = tmp_path / f"r_{swapped}.json"
                    lab = tmp_path / f"l_{swapped}.txt"
                    rc = cli.main(["run", "--input", path, *v, "--labels-out", str(lab), "-o", str(rep)])
                    outs.append((rc, _strip_timing(json.loads(rep.read_text())), lab.read_text()))
            assert outs[0] == outs[1], (name, v)
            assert outs[0][0] == 0


def test_reference_cli_frontier_and_ablation_identical(svcc_cli, tmp_path, monkeypatch):
    cli = svcc_cli
    files = _graphs(tmp_path, cli)
    for name, path in files.items():
        for sub, extra, drop in (("frontier", ["--threshold", "0.3"], {"elapsed"}),
                                 ("frontier", ["--kernel", "sparse-only"], {"elapsed"}),
                                 ("ablation", [], {"total_elapsed"})):
            outs = []
            for swapped in (False, True):
                with monkeypatch.context() as m:
                    if swapped:
                        _swap_to_b200(m, cli)
                    out = tmp_path / f"{sub}_{swapped}.csv"
                    rc = cli.main([sub, "--input", path, *extra, "-o", str(out)])
                    outs.append((rc, _csv_without(out, drop)))
            assert outs[0] == outs[1], (name, sub, extra)
