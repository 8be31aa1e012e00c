"""Dev tool: parity of one libfastsv variant on a few cases (vs the C oracle)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1910_05971_b200 import _native
_native.LIB_FASTSV_PATH = Path(sys.argv[1]).resolve()
import numpy as np
import oracle
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
case = sys.argv[2]
if case == "nccl":
    n, e = gen.rmat(13, 16, seed=21)
else:
    n, e = gen.baseline_graph(int(case[-1]))
g = fb.build_csr(n, e)
o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices)
for hubs in ((0, -1) if case != "nccl" else (-1, 0)):
    for mode in ("graph", "batch1", "nccl") if case == "nccl" else ("graph", "batch1"):
        s = fb.Solver(0, hub_slots=hubs)
        if mode == "nccl":
            s.attach_nccl(fb.Solver.nccl_unique_id(), 1, 0)
        s.upload(g)
        labels, iters, gfc, fc, ms, _ = s.run(batch=1 if mode == "batch1" else 0)
        ok = iters == o.iterations and gfc.tolist() == o.gf_changed.tolist() and np.array_equal(labels, o.labels)
        print(Path(sys.argv[1]).stem, case, "hubs", hubs, mode, "OK" if ok else f"FAIL iters {iters} vs {o.iterations} gfc {gfc.tolist()} vs {o.gf_changed.tolist()}", flush=True)
        s.close()
