"""Dev tool: raw edge list -> labels. Device CSR build (fsv_upload_edges)
vs host build_csr + fsv_upload_csr, for one BASELINE config.

    python tools/edges_time.py <config> [--check]
"""
import json
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen

cfg = int(sys.argv[1])
check = "--check" in sys.argv
out = {"config": cfg}
n, pairs = gen.baseline_graph(cfg)
out["n"], out["edges"] = n, int(pairs.shape[0])
pin = torch.from_numpy(pairs).pin_memory().numpy()        # pinned host pairs
s = fb.Solver(0)
ts = []
for _ in range(3):
    t = time.perf_counter(); s.upload_edges(n, pin); ts.append(time.perf_counter() - t)
out["upload_edges_s"] = [round(x, 4) for x in ts]
out["m_dir"] = s.m
st = s.solve()
out["solve_ms"] = round(st.solve_ms, 3)
lab = s.labels()
out["labels_digest"] = gen.pairs_digest(lab)
if check:
    g_dev = s.csr()
    t = time.perf_counter(); h = fb.build_csr(n, pairs); out["host_build_csr_s"] = round(time.perf_counter() - t, 2)
    out["csr_equal"] = bool(np.array_equal(g_dev.row_offsets, h.row_offsets)
                            and np.array_equal(g_dev.col_indices, h.col_indices))
    del g_dev
    t = time.perf_counter(); s.upload(h); out["host_csr_upload_s"] = round(time.perf_counter() - t, 3)
    s.solve()
    out["labels_equal"] = bool(np.array_equal(s.labels(), lab))
print(json.dumps(out), flush=True)
