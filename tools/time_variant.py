"""Dev tool: time one libfastsv variant on configs (best of 5 solves) and
check it against the reference-made golden record of each config."""
import json
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1910_05971_b200 import _native
_native.LIB_FASTSV_PATH = Path(sys.argv[1]).resolve()
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
golden = json.loads((ROOT / "tests" / "golden" / "configs.json").read_text())
out = []
for cfg in [int(c) for c in sys.argv[2:]]:
    n, pairs = gen.baseline_graph(cfg)
    g = fb.build_csr(n, pairs)
    s = fb.Solver(0)
    s.upload(g)
    ts = []
    best_it = None
    for _ in range(6):
        st = s.solve()
        ts.append(st.solve_ms)
        if st.solve_ms == min(ts):
            best_it = s.trace()[2].tolist()
    pr = s.solve(profile=True)
    prof = (pr.hook_ms / max(pr.hook_launches, 1) * 1e3, pr.push_ms * 1e3, pr.hubfix_ms * 1e3, pr.shortcut_ms * 1e3)
    ok = "n/a"
    rec = golden.get(str(cfg))
    if rec:
        labels, iters, gfc, fc, _, _ = s.run()
        ok = "OK" if (iters == rec["iterations"] and gfc.tolist() == rec["gf_changed"]
                      and fc.tolist() == rec["f_changed"]
                      and gen.pairs_digest(labels) == rec["labels_digest"]) else "PARITY-FAIL"
    out.append(f"cfg{cfg} {min(ts[1:]):.3f} ms (hook %.0f us avg, push %.0f us, hubfix %.0f us, sc %.0f us)" % prof + f" {ok} per-iter us {[round(x * 1e3) for x in best_it]}")
    s.close()
print(Path(sys.argv[1]).stem, " | ".join(out), flush=True)
