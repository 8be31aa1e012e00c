"""Dev tool: build one config and run a few solves (for ncu captures)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
cfg = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n, pairs = gen.baseline_graph(cfg)
g = fb.build_csr(n, pairs)
s = fb.Solver(0)
s.upload(g)
for _ in range(reps):
    st = s.solve(profile=len(sys.argv) > 3)
print("iters", st.iterations, "ms", st.solve_ms)
