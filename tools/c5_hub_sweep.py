"""Dev tool: config 5 solve time vs hub-table size (device edge build)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
n, pairs = gen.baseline_graph(5)
pin = torch.from_numpy(pairs).pin_memory().numpy()
for H in [int(x) for x in sys.argv[1:]] or [24576, 32768, 40960, 47104]:
    s = fb.Solver(0, hub_slots=H)
    s.upload_edges(n, pin)
    ts = [s.solve().solve_ms for _ in range(4)]
    pr = s.solve(profile=True)
    print(f"H={H} HT={s.stats.hub_slots} best {min(ts[1:]):.2f} ms hook {pr.hook_ms:.2f} first {pr.first_ms:.2f} push {pr.push_ms:.2f} sc {pr.shortcut_ms:.2f}", flush=True)
    s.close()
