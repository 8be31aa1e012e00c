"""Dev tool: exercise every device path on small graphs (for compute-sanitizer)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
from golden_io import load_suite
suite = load_suite()
s = fb.Solver(0)
bad = 0
for c in suite[::6]:
    g = fb.build_csr(c.n, c.edges)
    for hubs in (0, 256):
        s.set_hub_slots(hubs)
        s.upload(g)
        for policy, thr in ((0, 0.1), (2, 0.1), (3, 1.0)):
            lab, it, gfc, fc, ms, snaps = s.run(snapshots=False, policy=policy, threshold=thr)
            bad += (it != c.iterations) or not np.array_equal(lab, c.labels)
        lab, it, gfc, fc, ms, snaps = s.run(snapshots=True, snap_cap=64)
        bad += not np.array_equal(snaps, c.snapshots)
n, e = gen.rmat(12, 16, seed=3)
g = fb.build_csr(n, e)
s.set_hub_slots(0)
s.upload(g)
for policy in (0, 1, 2):
    s.run(policy=policy)
    s.run(batch=1, policy=policy)
lo, hi = 0, n // 2
s.upload(g, lo, hi, g.col_indices[g.row_offsets[lo]:g.row_offsets[hi]])
s.run()
print("sanitize run (single context) done, mismatches:", bad)
# device-CSR upload (borrowed arrays), tiled layouts, emulated rank groups
# with the delta exchange, and the device Labeling, all under the checks
import os
import torch
from paper_1910_05971_b200.driver import group_run
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench
n, e = gen.rmat(13, 16, seed=5)
g = fb.build_csr(n, e)
ref_lab = None
s.set_hub_slots(0)
s.upload(g)
ref_lab, ref_it = s.run()[:2]
d_off = torch.from_numpy(np.ascontiguousarray(g.row_offsets).copy()).cuda()
d_cols = torch.from_numpy(np.ascontiguousarray(g.col_indices).copy()).cuda()
s.upload_device(n, d_off.data_ptr(), d_cols.data_ptr())
lab, it = s.run()[:2]
bad += (it != ref_it) or not np.array_equal(lab, ref_lab)
lbl = s.labeling()
bad += not np.array_equal(lbl.labels, ref_lab.astype(np.int64))
for w in ("97", "1000"):
    os.environ["FSV_TILE_W"] = w
    for hubs in (-1, 0):
        s.set_hub_slots(hubs)
        s.upload(g)
        lab, it = s.run()[:2]
        bad += (it != ref_it) or not np.array_equal(lab, ref_lab)
del os.environ["FSV_TILE_W"]
for ranks in (2, 3):
    solvers = []
    for r in range(ranks):
        lo, hi = bench.row_partition(g.row_offsets, ranks, r)
        x = fb.Solver(0)
        x.upload(g, lo, hi, g.col_indices[g.row_offsets[lo]:g.row_offsets[hi]])
        solvers.append(x)
    for policy in (0, 2):
        lab, it = group_run(solvers, policy=policy)[:2]
        bad += (it != ref_it) or not np.array_equal(lab, ref_lab)
    for x in solvers:
        x.close()
print("sanitize run (device upload, tiles, groups) done, mismatches:", bad)
