"""Golden digests of the REFERENCE's CsrGraph (svcc.build_csr, graph.py:55-97)
for the device CSR build (fsv_upload_edges). Run here, where the reference
is importable (it is not on the GPU box):

    python tests/golden/make_csr_golden.py

Writes tests/golden/csr_digests.json: for every golden-suite graph and for
BASELINE configs 1 and 3 (the others take minutes in the reference's
np.unique-based build), n, m_dir and a digest of (row_offsets, col_indices)
as int64 little-endian bytes — the same bytes tests/golden_io.csr_digest
hashes on the device side.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

import svcc  # noqa: E402  (the reference)

from golden_io import csr_digest, load_suite  # noqa: E402
from paper_1910_05971_b200 import generators as gen  # noqa: E402


def record(n, edges):
    g = svcc.build_csr(n, edges)
    return {"n": int(n), "m_dir": int(g.m), "digest": csr_digest(g.row_offsets, g.col_indices)}


def main():
    path = HERE / "csr_digests.json"
    if len(sys.argv) > 2 and sys.argv[1] == "--configs":
        # add (or refresh) BASELINE configs only, keeping the rest:
        #   python tests/golden/make_csr_golden.py --configs 2 4   (minutes each)
        out = json.loads(path.read_text())
        for index in map(int, sys.argv[2:]):
            t = time.time()
            n, pairs = gen.baseline_graph(index)
            out["configs"][str(index)] = dict(record(n, pairs), pairs_digest=gen.pairs_digest(pairs))
            print(f"config {index}: reference build_csr {time.time() - t:.1f} s", flush=True)
        path.write_text(json.dumps(out, indent=0) + "\n")
        return
    out = {"suite": {}, "configs": {}}
    for c in load_suite():
        out["suite"][c.name] = record(c.n, c.edges.reshape(-1, 2))
    for index in (1, 3):
        t = time.time()
        n, pairs = gen.baseline_graph(index)
        out["configs"][str(index)] = dict(record(n, pairs), pairs_digest=gen.pairs_digest(pairs))
        print(f"config {index}: reference build_csr {time.time() - t:.1f} s", flush=True)
    path.write_text(json.dumps(out, indent=0) + "\n")
    print(f"{len(out['suite'])} suite graphs, configs {list(out['configs'])}")


if __name__ == "__main__":
    main()
