"""Dev tool: solve time vs hub-table size on a config."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n, pairs = gen.baseline_graph(cfg)
g = fb.build_csr(n, pairs)
for H in (24576, 32768, 40960, 47104, 49152, 51200, 53248, 57344):
    s = fb.Solver(0, hub_slots=H)
    s.upload(g)
    ts = [s.solve().solve_ms for _ in range(5)]
    pr = s.solve(profile=True)
    print(f"H={H:6d} used={s.stats.hub_slots:6d} solve {min(ts):.3f} ms  hook {pr.hook_ms*1e3:.0f} us  push {pr.push_ms*1e3:.0f} us", flush=True)
    s.close()
