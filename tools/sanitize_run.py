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
print("sanitize run done, mismatches:", bad)
