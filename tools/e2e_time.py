"""Dev tool: the bench's e2e loop (pinned host CSR -> upload -> solve ->
labels) with per-call timings, for one libfastsv build."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1910_05971_b200 import _native
if len(sys.argv) > 1:
    _native.LIB_FASTSV_PATH = Path(sys.argv[1]).resolve()
import numpy as np, torch
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
n, pairs = gen.baseline_graph(2)
g = fb.build_csr(n, pairs)
s = fb.Solver(0)
st = torch.cuda.current_stream()
s.set_stream(st.cuda_stream)
s.upload(g)
s.solve()
off = torch.from_numpy(np.ascontiguousarray(g.row_offsets).copy()).pin_memory()
cols = torch.from_numpy(np.ascontiguousarray(g.col_indices).copy()).pin_memory()
lab = torch.empty(n, dtype=torch.int32).pin_memory()
for rep in range(5):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    ev[0].record(st)
    s.upload_arrays(n, off.data_ptr(), cols.data_ptr(), 0, n)
    t1 = time.perf_counter()
    ev[1].record(st)
    s.solve()
    t2 = time.perf_counter()
    ev[2].record(st)
    s.labels_into(lab.data_ptr())
    ev[3].record(st)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(Path(sys.argv[1]).stem if len(sys.argv) > 1 else "lib",
          "dev ms upload %.2f solve %.2f labels %.2f | host ms upload %.2f solve %.2f total %.2f" % (
          ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]),
          (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t0) * 1e3), flush=True)
