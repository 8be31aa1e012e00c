"""Dev tool: e2e upload timing (pinned buffers) vs the pure H2D copy."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_1910_05971_b200 import _native
if len(sys.argv) > 1:
    _native.LIB_FASTSV_PATH = Path(sys.argv[1]).resolve()
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
n, pairs = gen.baseline_graph(2)
g = fb.build_csr(n, pairs)
off = torch.from_numpy(np.ascontiguousarray(g.row_offsets).copy()).pin_memory()
cols = torch.from_numpy(np.ascontiguousarray(g.col_indices).copy()).pin_memory()
s = fb.Solver(0)
st = torch.cuda.current_stream()
s.set_stream(st.cuda_stream)
def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts[1:])
up = timed(lambda: s.upload_arrays(n, off.data_ptr(), cols.data_ptr()))
sol = timed(lambda: s.solve())
d_off = torch.empty_like(off, device="cuda"); d_cols = torch.empty_like(cols, device="cuda")
def cp():
    d_off.copy_(off, non_blocking=True); d_cols.copy_(cols, non_blocking=True)
h2d = timed(cp)
print(f"{Path(sys.argv[1]).stem if len(sys.argv) > 1 else ''} chunks={os.environ.get('FSV_UPLOAD_CHUNKS','default')} upload {up:.2f} ms  solve {sol:.3f} ms  pure H2D {h2d:.2f} ms")
