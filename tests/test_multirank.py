"""N>1 path on CPU: two gloo ranks, each owning a 1D row partition balanced
by entries (bench.row_partition), run the emulated device
schedule with a real torch.distributed all_reduce(MIN) standing in for the
library's ncclAllReduce(ncclInt32, ncclMin). Snapshots must equal the
single-device reference run (E4)."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import emulate
        import paper_1910_05971_b200 as fb
        from golden_io import load_suite
        from paper_1910_05971_b200 import generators as gen

        def allreduce_min(a):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64))
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            return t.numpy()

        def allgather_pairs(pairs):
            # the library's protocol: one allgather of the counts, then one of
            # the (index, value) lists padded to the largest
            cnt = torch.tensor([len(pairs)], dtype=torch.int64)
            counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(counts, cnt)
            cmax = max(int(c.item()) for c in counts)
            buf = torch.zeros((max(cmax, 1), 2), dtype=torch.int64)
            buf[:len(pairs)] = torch.from_numpy(pairs)
            outs = [torch.zeros_like(buf) for _ in range(world)]
            dist.all_gather(outs, buf)
            return [o[:int(c.item())].numpy() for o, c in zip(outs, counts)]

        results = []
        cases = [(c.name, c.n, c.edges) for c in load_suite()[::9]]
        n, e = gen.rmat(11, 16, seed=9)
        cases.append(("rmat11", n, e))
        for name, n, edges in cases:
            g = fb.build_csr(n, edges)
            lo, hi = bench.row_partition(g.row_offsets, world, rank)
            f, it, gfc, fc, snaps = emulate.run(n, g.row_offsets, g.col_indices, lo, hi, allreduce_min)
            results.append((name, it, gfc, fc, np.stack(snaps) if snaps else None))
            # the same with the sparse-iteration delta exchange
            st = {}
            f, it, gfc, fc, snaps = emulate.run(n, g.row_offsets, g.col_indices, lo, hi, allreduce_min,
                                                allgather_pairs=allgather_pairs, nranks=world, stats=st)
            results.append((name + "#delta", it, gfc, fc, np.stack(snaps) if snaps else None, st))
        if rank == 0:
            q.put(results)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_schedule_matches_single_device():
    sys.path.insert(0, str(ROOT / "tests"))
    import emulate
    import oracle
    import paper_1910_05971_b200 as fb
    from golden_io import load_suite
    from paper_1910_05971_b200 import generators as gen

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    golden = {c.name: c for c in load_suite()}
    deltas = 0
    for rec in results:
        name, it, gfc, fc, snaps = rec[:5]
        if name.endswith("#delta"):
            deltas += rec[5].get("delta", 0)
            name = name[:-len("#delta")]
        if name in golden:
            c = golden[name]
            assert it == c.iterations and gfc == c.gf_changed and fc == c.f_changed, name
            assert np.array_equal(snaps, c.snapshots), name
        else:
            n, e = gen.rmat(11, 16, seed=9)
            g = fb.build_csr(n, e)
            o = oracle.fastsv_csr(n, g.row_offsets, g.col_indices, snapshots=True)
            assert it == o.iterations and gfc == o.gf_changed.tolist(), name
            assert np.array_equal(snaps, o.snapshots), name
    assert deltas > 0, "no sparse iteration took the delta exchange"


def test_row_partition_covers_rows_and_balances_entries():
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_1910_05971_b200 as fb
    from paper_1910_05971_b200 import generators as gen
    n, e = gen.rmat(12, 16, seed=2)
    g = fb.build_csr(n, e)
    for world in (1, 2, 4, 8):
        parts = [bench.row_partition(g.row_offsets, world, r) for r in range(world)]
        assert parts[0][0] == 0 and parts[-1][1] == n
        for (a, b), (c, d) in zip(parts, parts[1:]):
            assert b == c
        sizes = [g.row_offsets[b] - g.row_offsets[a] for a, b in parts]
        assert sum(sizes) == g.m
        assert max(sizes) <= g.m / world + g.degrees.max() + 1
