"""Dev tool: config 5 solve time for one libfastsv build (device edge build)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1910_05971_b200 import _native
_native.LIB_FASTSV_PATH = Path(sys.argv[1]).resolve()
import torch
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
n, pairs = gen.baseline_graph(5)
pin = torch.from_numpy(pairs).pin_memory().numpy()
s = fb.Solver(0)
s.upload_edges(n, pin)
ts = [s.solve().solve_ms for _ in range(4)]
st = s.stats
pr = s.solve(profile=True)
lab = s.labels()
print(Path(sys.argv[1]).stem, "HT", st.hub_slots, "best %.2f ms" % min(ts[1:]), "hook %.2f first %.2f push %.2f hubfix %.2f sc %.2f" %
      (pr.hook_ms, pr.first_ms, pr.push_ms, pr.hubfix_ms, pr.shortcut_ms), "labels", gen.pairs_digest(lab), flush=True)
