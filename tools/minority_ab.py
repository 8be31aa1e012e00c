"""Dev tool: per-iteration times with the minority sweep on and off."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n, pairs = gen.baseline_graph(cfg)
g = fb.build_csr(n, pairs)
s = fb.Solver(0)
s.upload(g)
for on in (True, False, True, False):
    s.set_minority_sweep(on)
    best = None
    for _ in range(6):
        st = s.solve()
        it = [round(x * 1e3) for x in s.trace()[2].tolist()]
        if best is None or st.solve_ms < best[0]:
            best = (st.solve_ms, it)
    pr = s.solve(profile=True)
    print(f"minority={on} best {best[0]:.3f} ms per-iter us {best[1]} | profile: hook {pr.hook_ms*1e3:.0f} us over {pr.hook_launches} dense launches, push {pr.push_ms*1e3:.0f}, sc {pr.shortcut_ms*1e3:.0f}", flush=True)
