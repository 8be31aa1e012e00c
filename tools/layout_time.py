"""Dev tool: layout build time from a device-resident CSR (fsv_upload_csr_device),
best of N uploads, for a libfastsv build.   python tools/layout_time.py <lib.so> <config> [reps]"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1910_05971_b200 import _native
_native.LIB_FASTSV_PATH = Path(sys.argv[1]).resolve()
import numpy as np
import torch
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
cfg = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
n, pairs = gen.baseline_graph(cfg)
g = fb.build_csr(n, pairs)
del pairs
s = fb.Solver(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); s.set_stream(st.cuda_stream)
d_off = torch.from_numpy(np.ascontiguousarray(g.row_offsets).copy()).cuda()
d_cols = torch.from_numpy(np.ascontiguousarray(g.col_indices).copy()).cuda()
ts = []
for _ in range(reps):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); s.upload_device(n, d_off.data_ptr(), d_cols.data_ptr()); b.record(st)
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
r = s.solve()
lab = s.labels()
print(Path(sys.argv[1]).stem, f"cfg{cfg} layout best {min(ts[1:]):.3f} ms (all {[round(x, 3) for x in ts]}) solve {r.solve_ms:.3f} "
      f"iters {r.iterations} E {r.oriented_entries} labels {gen.pairs_digest(lab)}", flush=True)
