"""Dev tool: one libfastsv build on one config: oriented entries, iterations,
labels digest, best solve and per-phase times.

    python tools/layout_check.py <lib.so> <config>
"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1910_05971_b200 import _native
_native.LIB_FASTSV_PATH = Path(sys.argv[1]).resolve()
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
n, pairs = gen.baseline_graph(int(sys.argv[2]))
g = fb.build_csr(n, pairs)
s = fb.Solver(0)
s.upload(g)
ts = [s.solve().solve_ms for _ in range(6)]
st = s.stats
pr = s.solve(profile=True)
lab = s.labels()
print(Path(sys.argv[1]).stem, "E", st.oriented_entries, "iters", st.iterations, "best %.3f" % min(ts[1:]),
      "hook %.1f us/%d push %.1f sc %.1f hubfix %.1f" % (pr.hook_ms * 1e3, pr.hook_launches, pr.push_ms * 1e3,
                                                      pr.shortcut_ms * 1e3, pr.hubfix_ms * 1e3),
      "labels", gen.pairs_digest(lab), flush=True)
