"""Accessors for the reference-produced golden vectors (tests/golden/)."""

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@dataclass
class GoldenCase:
    name: str
    n: int
    m_dir: int
    edges: np.ndarray          # raw int32 pairs (k, 2)
    iterations: int
    gf_changed: list
    f_changed: list
    labels: np.ndarray         # int32
    snapshots: np.ndarray      # (iterations, n) int32


def load_suite():
    d = np.load(GOLDEN / "suite.npz", allow_pickle=False)
    out = []
    for i, name in enumerate(d["names"]):
        n = int(d["n"][i])
        e = d["edges"][d["edge_off"][i]:d["edge_off"][i + 1]].reshape(-1, 2)
        t0, t1 = d["trace_off"][i], d["trace_off"][i + 1]
        it = int(d["iterations"][i])
        lab_off = int(d["n"][:i].sum())
        s0, s1 = d["snap_off"][i], d["snap_off"][i + 1]
        out.append(GoldenCase(str(name), n, int(d["m_dir"][i]), e, it,
                              d["gf_changed"][t0:t1].tolist(), d["f_changed"][t0:t1].tolist(),
                              d["labels"][lab_off:lab_off + n], d["snapshots"][s0:s1].reshape(it, n)))
    return out


def load_configs():
    return {int(k): v for k, v in json.loads((GOLDEN / "configs.json").read_text()).items()}


def load_kats():
    return json.loads((GOLDEN / "kats.json").read_text())


def load_driver_traces():
    """{(config_name, graph_name): (kernel list, flops list)} from the reference."""
    d = np.load(GOLDEN / "driver_traces.npz", allow_pickle=False)
    out = {}
    for i, nm in enumerate(d["names"]):
        cfg, name = str(nm).split(":", 1)
        a, b = d["off"][i], d["off"][i + 1]
        out[(cfg, name)] = (d["kernel"][a:b].tolist(), d["flops"][a:b].tolist())
    return out


def csr_digest(row_offsets, col_indices) -> str:
    """sha256 (first 16 hex) of a CSR as int64 little-endian bytes: offsets, then columns."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(row_offsets, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(col_indices, dtype="<i8").tobytes())
    return h.hexdigest()[:16]


def load_csr_digests():
    return json.loads((GOLDEN / "csr_digests.json").read_text())


def load_variants():
    """Reference traces of the hooking variants: list of (graph name, code,
    iterations, gf_changed, f_changed, snapshot digest) and the pair-stream
    digests of the generated extra graphs."""
    d = np.load(GOLDEN / "variants.npz", allow_pickle=False)
    runs = []
    for i in range(len(d["names"])):
        a, b = d["trace_off"][i], d["trace_off"][i + 1]
        runs.append((str(d["names"][i]), int(d["codes"][i]), int(d["iterations"][i]),
                     d["gf_changed"][a:b].tolist(), d["f_changed"][a:b].tolist(), str(d["digests"][i])))
    extra = dict(zip([str(x) for x in d["extra_names"]], [str(x) for x in d["extra_digests"]]))
    return runs, extra


def variant_graphs():
    """{name: (n, pairs)} for every graph of the variant goldens (the suite
    plus the generated extras, regenerated from the same seeded streams)."""
    from paper_1910_05971_b200 import generators as gen
    out = {c.name: (c.n, c.edges) for c in load_suite()}
    out["x:config1"] = gen.baseline_graph(1)
    out["x:rmat14"] = gen.rmat(14, 16, seed=5)
    out["x:grid300"] = gen.grid(300, 300, 0.4, seed=3)
    out["x:forest2000"] = gen.forest(2000, 1, 64, 2, seed=4)
    return out
