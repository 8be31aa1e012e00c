"""Dev tool: config graph -> device CSR (torch) -> layout (fsv_upload_csr_device)
-> solves; for ncu captures and layout/solve timing.

    python tools/prof_solve.py [--config 2] [--reps 3] [--profile] [--uploads 2]
"""
import argparse
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--scale", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--uploads", type=int, default=2)
ap.add_argument("--profile", action="store_true")
a = ap.parse_args()
n, pairs = gen.baseline_graph(a.config, a.scale)
g = fb.build_csr(n, pairs)
del pairs
s = fb.Solver(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
s.set_stream(st.cuda_stream)
d_off = torch.from_numpy(np.ascontiguousarray(g.row_offsets)).cuda()
d_cols = torch.from_numpy(np.ascontiguousarray(g.col_indices)).cuda()
for u in range(a.uploads):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.upload_device(n, d_off.data_ptr(), d_cols.data_ptr())
    e1.record(st)
    torch.cuda.synchronize()
    print(f"upload {u}: {e0.elapsed_time(e1):.3f} ms", flush=True)
for _ in range(a.reps):
    try:
        r = s.solve(profile=a.profile)
    except Exception as e:      # dev probes with broken semantics may not converge
        print("solve failed:", e)
        break
    print(f"solve {r.solve_ms:.3f} ms iters {r.iterations} hook {r.hook_ms:.3f} ({r.hook_launches}) push {r.push_ms:.3f} "
          f"first {r.first_ms:.3f} shortcut {r.shortcut_ms:.3f}", flush=True)
