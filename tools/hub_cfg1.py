"""Dev tool: config 1 (and small RMATs) solve time vs hub-table setting."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
cases = [("cfg1", gen.baseline_graph(1)), ("rmat14", gen.rmat(14, 16, seed=1)), ("rmat16", gen.rmat(16, 16, seed=1)),
         ("rmat18", gen.rmat(18, 16, seed=1)), ("rmat20", gen.rmat(20, 16, seed=1))]
for name, (n, e) in cases:
    g = fb.build_csr(n, e)
    out = []
    for hubs in (0, -1, 1024, 8192):
        s = fb.Solver(0, hub_slots=hubs)
        s.upload(g)
        ts = [s.solve().solve_ms for _ in range(8)]
        out.append(f"hubs {hubs}: {min(ts[2:]):.3f} ms (H={s.stats.hub_slots})")
        s.close()
    print(name, "n", n, " | ".join(out), flush=True)
