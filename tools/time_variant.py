"""Dev tool: time one libfastsv variant on configs (best of 5 solves)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1910_05971_b200 import _native
_native.LIB_FASTSV_PATH = Path(sys.argv[1]).resolve()
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
out = []
for cfg in [int(c) for c in sys.argv[2:]]:
    n, pairs = gen.baseline_graph(cfg)
    g = fb.build_csr(n, pairs)
    s = fb.Solver(0)
    s.upload(g)
    ts = [s.solve().solve_ms for _ in range(6)]
    pr = s.solve(profile=True)
    out.append(f"cfg{cfg} {min(ts[1:]):.3f} ms (hook {pr.hook_ms/max(pr.hook_launches,1)*1e3:.0f} us avg, sc {pr.shortcut_ms*1e3:.0f} us)")
    s.close()
print(Path(sys.argv[1]).stem, " | ".join(out), flush=True)
