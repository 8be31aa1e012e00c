"""Dev tool (this container only: imports the reference from /root/reference):
time svcc.fastsv_la against the numpy port (oracle/port.py) on RMAT-20."""
import sys, time, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/reference/pkg/src')
import numpy as np
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
from oracle import port
import svcc
from svcc.graph import CsrGraph
n, pairs = gen.rmat(20, 16, seed=0)
g = fb.build_csr(n, pairs)
off = np.asarray(g.row_offsets, dtype=np.int64); cols = np.asarray(g.col_indices, dtype=np.int64)
try:
    rg = CsrGraph(n=n, row_offsets=off, col_indices=cols)
except TypeError:
    rg = CsrGraph(n, off, cols)
cores = len(os.sched_getaffinity(0))
for w in (1, cores):
    t = time.time(); r = svcc.fastsv_la(rg, svcc.DriverConfig(workers=w)); tr = time.time() - t
    pg = port.PortGraph(n, off, cols)
    t = time.time(); f, it, gfc, kinds = port.fastsv_la(pg, workers=w); tp = time.time() - t
    print("workers", w, "reference %.2f s" % tr, "port %.2f s" % tp, "iters", r.iterations, it, flush=True)
