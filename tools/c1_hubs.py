import sys; sys.path.insert(0, '/root/repo')
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
n, pairs = gen.baseline_graph(1)
g = fb.build_csr(n, pairs)
for hubs in (-1, 0, 1024, 4096):
    s = fb.Solver(0, hub_slots=hubs); s.upload(g)
    ts = [s.solve().solve_ms for _ in range(8)]
    st = s.stats
    print("hubs", hubs, "H", st.hub_slots, "best %.3f ms" % min(ts[2:]), "per-iter", [round(x*1e3) for x in s.trace()[2].tolist()], flush=True)
    s.close()
