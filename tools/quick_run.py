"""Dev tool: generate a BASELINE config, solve on the GPU, compare with the
C oracle, print per-iteration device times."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import oracle
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen

cfgs = [int(a) for a in sys.argv[1:]] or [1, 2]
for c in cfgs:
    t = time.time(); n, pairs = gen.baseline_graph(c); tg = time.time() - t
    t = time.time(); g = fb.build_csr(n, pairs); tb = time.time() - t
    print(f"config {c}: n={n} m={len(pairs)} m_dir={g.m} gen {tg:.1f}s csr {tb:.1f}s", flush=True)
    for hubs in (0, -1):
        s = fb.Solver(0, hub_slots=hubs)
        t = time.time(); s.upload(g); tu = time.time() - t
        times = []
        for rep in range(6):
            st = s.solve()
            times.append(st.solve_ms)
        pr = s.solve(profile=True)
        print(f"  profile: first {pr.first_ms*1e3:.1f} us  hook {pr.hook_ms*1e3:.1f} us/{pr.hook_launches}  hubfix {pr.hubfix_ms*1e3:.1f} us  push {pr.push_ms*1e3:.1f} us ({pr.sparse_iterations} sparse)  shortcut {pr.shortcut_ms*1e3:.1f} us  total {pr.solve_ms*1e3:.1f} us")
        lab = s.labels()
        gfc, fc, ms = s.trace()
        print(f"  hubs={st.hub_slots} E={st.oriented_entries} upload {tu*1e3:.0f} ms  iters {st.iterations} "
              f"solve ms {['%.3f' % x for x in times]}  syncs {st.host_syncs} launches {st.kernel_launches}")
        print(f"  per-iter ms {['%.3f' % x for x in ms]}  gfc {gfc.tolist()}")
        s.close()
    t = time.time(); o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices); to = time.time() - t
    ok = o.iterations == st.iterations and np.array_equal(o.labels, lab) and o.gf_changed.tolist() == gfc.tolist() and o.f_changed.tolist() == fc.tolist()
    print(f"  oracle {to:.1f}s iters {o.iterations} gfc {o.gf_changed.tolist()} PARITY {'OK' if ok else 'FAIL'}", flush=True)
    best = min(times) / 1e3
    print(f"  edges/s {len(pairs)/best:.3e}  B_iter-model frac {(o.iterations*(4*g.m + 4*(n+1) + 24*n))/best/6553.3e9:.3f}")
