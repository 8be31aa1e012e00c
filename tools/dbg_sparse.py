"""Dev tool: phase timing of the sparse k_hook path (debug build)."""
import ctypes, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
from paper_1910_05971_b200 import _native
dbg = ROOT / "paper_1910_05971_b200" / "libfastsv_dbg.so"
_native.LIB_FASTSV_PATH = dbg
lib = _native.fastsv_lib()
lib.fsv_debug_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
n, pairs = gen.baseline_graph(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
g = fb.build_csr(n, pairs)
s = fb.Solver(0)
s.upload(g)
for rep in range(3):
    st = s.solve(batch=1, max_iters=0)
print("iters", st.iterations, "ms", st.solve_ms, "sparse", st.sparse_iterations)
t = np.zeros(148 * 4, dtype=np.uint64)
lib.fsv_debug_timing(t.ctypes.data, t.size)
t = t.reshape(148, 4).astype(np.int64)
t0 = t[:, 0].min()
print("start spread us", (t[:, 0].max() - t0) / 1e3)
print("phase1 end (us) min/med/max", np.percentile((t[:, 1] - t0) / 1e3, [0, 50, 100]))
print("barrier release (us) min/max", (t[:, 2].min() - t0) / 1e3, (t[:, 2].max() - t0) / 1e3)
print("phase2 end (us) min/med/max", np.percentile((t[:, 3] - t0) / 1e3, [0, 50, 100]))
