"""CLI contract (cli.py of the reference, pkg/tests/test_cli.py as the model):
subcommands, file formats, report schemas, exit codes. Input and usage
errors are checked on CPU (they fail before the device is touched); runs
are GPU tests."""

import csv
import json

import numpy as np
import pytest

import oracle
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import cli

TWO_TRIANGLES_MM = ("%%MatrixMarket matrix coordinate pattern symmetric\n"
                    "6 6 6\n2 1\n3 2\n3 1\n5 4\n6 5\n6 4\n")


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def path_edges(tmp_path, n, name="path.el"):
    return write(tmp_path, name, "".join(f"{i} {i + 1}\n" for i in range(n - 1)))


def read_csv(path):
    with open(path, newline="") as fh:
        return list(csv.reader(fh))


# ---- CPU: readers, usage errors, the independent verifier -------------------

def test_read_matrix_market_and_edge_list(tmp_path):
    g = cli.load_graph(write(tmp_path, "t.mtx", TWO_TRIANGLES_MM))
    assert g.n == 6 and g.m == 12
    assert g.row_offsets.tolist() == [0, 2, 4, 6, 8, 10, 12]
    e = cli.load_graph(write(tmp_path, "t.el", "# comment\n0 1\n\n1 2\n4 4\n"))
    assert e.n == 5 and e.m == 4                          # self-loop keeps vertex 4
    assert cli.load_graph(write(tmp_path, "empty.el", "")).n == 0
    gen_mm = ("%%MatrixMarket matrix coordinate real general\n% c\n3 3 2\n1 2 0.5\n3 3 1.0\n")
    assert cli.load_graph(write(tmp_path, "g.mtx", gen_mm)).m == 2


@pytest.mark.parametrize("text,msg", [
    ("%%MatrixMarket matrix array real general\n2 2\n", "array"),
    ("%%MatrixMarket matrix coordinate complex general\n2 2 0\n", "unsupported field"),
    ("%%MatrixMarket matrix coordinate pattern hermitian\n2 2 0\n", "unsupported qualifier"),
    ("%%MatrixMarket matrix coordinate pattern general\n2 3 0\n", "must be square"),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 3\n", "out of bounds"),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n", "declares 2 entries, found 1"),
    ("%%MatrixMarket matrix coordinate pattern general\n", "missing dimension"),
])
def test_malformed_matrix_market(tmp_path, text, msg):
    with pytest.raises(fb.InputError, match=msg):
        cli.read_matrix_market(write(tmp_path, "bad.mtx", text))


def test_malformed_edge_list(tmp_path):
    for text, msg in (("0 1 2\n", "expected two ids at line 1"), ("0 x\n", "non-integer"),
                      ("0 -1\n", "negative id")):
        with pytest.raises(fb.InputError, match=msg):
            cli.read_edge_list(write(tmp_path, "bad.el", text))


def test_usage_and_input_errors_exit_1(tmp_path, capsys):
    p = write(tmp_path, "t.mtx", TWO_TRIANGLES_MM)
    assert cli.main(["run", "--input", str(tmp_path / "missing.el")]) == 1
    assert "error:" in capsys.readouterr().err
    assert cli.main(["run", "--input", p, "--bogus"]) == 1
    assert cli.main(["run", "--input", p, "--algo", "sv", "--sv-level", "2"]) == 1
    assert cli.main(["run", "--input", p, "--algo", "fastsv-la", "--hook-stochastic"]) == 1
    assert cli.main(["run", "--input", p, "--algo", "fastsv-la", "--threshold", "1.5"]) == 1
    assert cli.main(["frontier", "--input", p, "--threads", "0"]) == 1
    assert cli.main(["run", "--input", write(tmp_path, "b.mtx", "%%MatrixMarket x\n")]) == 1


def test_independent_verifier_matches_union_find():
    rng = np.random.default_rng(5)
    for n in (1, 7, 300):
        e = rng.integers(0, n, (n, 2))
        g = fb.build_csr(n, e)
        assert np.array_equal(cli.min_id_components(g), oracle.uf_labels(n, e).astype(np.int64))


# ---- GPU: the commands ------------------------------------------------------

@pytest.mark.gpu
def test_run_fastsv_la_two_triangles(tmp_path, capsys):
    p = write(tmp_path, "t.mtx", TWO_TRIANGLES_MM)
    assert cli.main(["run", "--input", p, "--algo", "fastsv-la", "--verify"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["graph"] == {"n": 6, "m": 12, "source": p}
    assert rep["algorithm"] == "fastsv-la" and rep["component_count"] == 2 and rep["verified"] is True
    assert rep["config"] == {"sparse_threshold": 0.1, "force_kernel": "auto", "workers": 1}
    assert len(rep["trace"]) == rep["iterations"]
    assert set(rep["trace"][0]) == {"iteration", "gf_changed", "f_changed", "kernel", "flops", "elapsed"}
    assert rep["trace"][-1]["gf_changed"] == 0


@pytest.mark.gpu
def test_run_sv_levels_and_flags(tmp_path, capsys):
    p = path_edges(tmp_path, 40)
    assert cli.main(["run", "--input", p, "--algo", "sv", "--verify"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["config"] == {} and rep["component_count"] == 1
    assert all(t["kernel"] == "none" for t in rep["trace"])
    assert cli.main(["run", "--input", p, "--algo", "fastsv", "--sv-level", "3"]) == 0
    cfg = json.loads(capsys.readouterr().out)["config"]
    assert cfg == {"grandparent_hooking": True, "stochastic_hooking": True, "aggressive_hooking": False,
                   "early_termination": False}
    assert cli.main(["run", "--input", p, "--algo", "fastsv", "--sv-level", "3", "--hook-aggressive"]) == 0
    assert json.loads(capsys.readouterr().out)["config"]["aggressive_hooking"] is True


@pytest.mark.gpu
def test_run_labels_out_and_report_file(tmp_path):
    p = write(tmp_path, "t.mtx", TWO_TRIANGLES_MM)
    out, lab = tmp_path / "r.json", tmp_path / "labels.txt"
    assert cli.main(["run", "--input", p, "--labels-out", str(lab), "-o", str(out)]) == 0
    assert lab.read_text().split("\n")[:6] == ["0 0", "1 0", "2 0", "3 3", "4 3", "5 3"]
    assert json.loads(out.read_text())["iterations"] >= 1


@pytest.mark.gpu
def test_verification_failure_exits_2(tmp_path, monkeypatch, capsys):
    p = write(tmp_path, "t.mtx", TWO_TRIANGLES_MM)
    monkeypatch.setattr(cli, "min_id_components", lambda g: np.zeros(g.n, dtype=np.int64))
    assert cli.main(["run", "--input", p, "--verify"]) == 2
    assert "verification failed" in capsys.readouterr().err


@pytest.mark.gpu
def test_invariant_violation_exits_3(tmp_path, monkeypatch, capsys):
    p = write(tmp_path, "t.mtx", TWO_TRIANGLES_MM)

    def broken(g, cfg=None):
        raise fb.InvariantError("algorithm terminated on non-star forest")
    monkeypatch.setattr(cli, "fastsv_la", broken)
    assert cli.main(["run", "--input", p, "--algo", "fastsv-la"]) == 3
    assert "invariant violated" in capsys.readouterr().err


@pytest.mark.gpu
def test_ablation_path64(tmp_path):
    out = tmp_path / "a.csv"
    assert cli.main(["ablation", "--input", path_edges(tmp_path, 64), "-o", str(out)]) == 0
    rows = read_csv(out)
    assert rows[0] == ["name", "iterations", "total_elapsed", "reduction_vs_sv1"]
    assert [r[0] for r in rows[1:]] == ["sv1", "sv2", "sv3", "sv4", "sv5"]
    assert rows[1][3] == "0.0000"
    assert int(rows[5][1]) <= int(rows[1][1])


@pytest.mark.gpu
def test_frontier_trace_and_kernel_choice(tmp_path):
    p = write(tmp_path, "t.mtx", TWO_TRIANGLES_MM)
    out = tmp_path / "f.csv"
    assert cli.main(["frontier", "--input", p, "-o", str(out)]) == 0
    rows = read_csv(out)
    assert rows[0] == ["iteration", "gf_changed", "gf_changed_frac", "kernel", "flops", "elapsed"]
    assert rows[1][3] == "dense" and rows[-1][1] == "0"
    assert cli.main(["frontier", "--input", p, "--kernel", "dense-only", "-o", str(out)]) == 0
    assert all(r[3] == "dense" for r in read_csv(out)[1:])
    assert cli.main(["frontier", "--input", p, "--threshold", "1.0", "-o", str(out)]) == 0
    kinds = [r[3] for r in read_csv(out)[1:]]
    assert kinds[0] == "dense" and all(k == "sparse" for k in kinds[1:])
