"""Golden record of BASELINE config 5 (RMAT-27, edgefactor 16: 2^31 pairs,
~4.2e9 directed CSR entries, int64 offsets) from the C ORACLE.

The Python reference cannot run config 5 (svcc.build_csr needs
~100 GB of int64 temporaries and union_find_labels is a pure-Python loop), so
the checker is oracle/fsv_oracle.c, whose restatements are pinned to the
reference itself on configs 1-4 and 379 golden graphs (tests/test_oracle.py):
  - union-find + min relabel (oracle.py:12-55) over the raw pairs -> labels;
  - all-flags FastSV, edge form (algorithms.py:79-91,117-142) over the
    symmetric CSR -> iteration count, gf_changed / f_changed per iteration,
    labels (must equal the union-find labels).
Needs ~60 GB of host memory and a few minutes of one core for each oracle;
run on a GPU-box host (it needs no GPU):

    python tests/golden/make_config5_golden.py > gpurun_out/config5_golden.json

then merge the printed record into tests/golden/configs.json["5"] with
    python tests/golden/make_config5_golden.py --merge gpurun_out/config5_golden.json
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))


def make():
    import oracle
    from paper_1910_05971_b200 import build_csr
    from paper_1910_05971_b200 import generators as gen
    rec = {"config": 5}
    t = time.time()
    n, pairs = gen.baseline_graph(5)
    rec.update(n=n, edges=int(pairs.shape[0]), pairs_digest=gen.pairs_digest(pairs),
               gen_s=round(time.time() - t, 1))
    t = time.time()
    uf = oracle.uf_labels(n, pairs)
    rec["uf_s"] = round(time.time() - t, 1)
    rec["uf_labels_digest"] = gen.pairs_digest(uf)
    t = time.time()
    g = build_csr(n, pairs)
    del pairs
    rec["m_dir"] = int(g.m)
    rec["csr_s"] = round(time.time() - t, 1)
    t = time.time()
    o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, cap=64)
    rec["oracle_fastsv_s"] = round(time.time() - t, 1)
    assert np.array_equal(o.labels, uf), "FastSV oracle labels differ from union-find"
    rec.update(iterations=int(o.iterations), gf_changed=o.gf_changed.tolist(), f_changed=o.f_changed.tolist(),
               component_count=int(np.count_nonzero(o.labels == np.arange(n, dtype=np.int32))),
               labels_digest=gen.pairs_digest(o.labels),
               checker="oracle/fsv_oracle.c (union-find + FastSV edge form); reference infeasible at this size")
    return rec


def main():
    if len(sys.argv) == 3 and sys.argv[1] == "--merge":
        text = Path(sys.argv[2]).read_text()
        rec = json.loads([ln for ln in text.splitlines() if ln.startswith("{")][-1])
        path = HERE / "configs.json"
        d = json.loads(path.read_text())
        d["5"] = rec
        path.write_text(json.dumps(d, indent=1) + "\n")
        print("merged config 5:", {k: rec[k] for k in ("iterations", "component_count", "labels_digest")})
        return
    print(json.dumps(make()), flush=True)


if __name__ == "__main__":
    main()
