"""Dev tool: API-level (torch events around Solver.solve) vs library device
time (events inside fsv_solve) for config 2, with the bench's L2 flush."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1910_05971_b200 as fb
from paper_1910_05971_b200 import generators as gen
n, pairs = gen.baseline_graph(2)
g = fb.build_csr(n, pairs)
s = fb.Solver(0)
st = torch.cuda.current_stream()
s.set_stream(st.cuda_stream)
s.upload(g)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty(1, dtype=torch.int64, device="cuda")
for flushed in (False, True):
    api, dev = [], []
    for i in range(25):
        if flushed:
            flush.zero_(); torch.sum(rd.view(torch.int64), dim=0, keepdim=True, out=sink)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); stt = s.solve(); b.record(st)
        torch.cuda.synchronize()
        if i >= 5:
            api.append(a.elapsed_time(b)); dev.append(stt.solve_ms)
    print("flushed" if flushed else "warm   ", "api %.3f ms  device %.3f ms" % (sum(api) / len(api), sum(dev) / len(dev)))
