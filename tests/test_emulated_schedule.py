"""The device schedule (oriented layout, closed-form iteration 1, filtered
row/column hooks, allreduce-min merge) emulated in numpy, single process:
identical snapshots to the reference on the golden suite (E1-E4)."""

import numpy as np

import emulate
import paper_1910_05971_b200 as fb
from golden_io import load_suite


def test_emulated_schedule_matches_reference():
    for c in load_suite():
        g = fb.build_csr(c.n, c.edges)
        f, it, gfc, fc, snaps = emulate.run(c.n, g.row_offsets, g.col_indices)
        assert it == c.iterations, c.name
        assert gfc == c.gf_changed and fc == c.f_changed, c.name
        assert np.array_equal(np.stack(snaps), c.snapshots), c.name


def test_partitioned_schedule_single_process():
    # P partitions merged by elementwise min == single device (E4)
    for c in load_suite()[::7]:
        g = fb.build_csr(c.n, c.edges)
        for P in (2, 3, 4):
            parts = []
            for r in range(P):
                lo, hi = c.n * r // P, c.n * (r + 1) // P
                parts.append((lo, hi))
            # run the P ranks in lock-step with an in-process "allreduce"
            states = {}

            def allreduce(a, _states=states):
                return a
            # emulate: every rank computes its contribution; merge via min
            rows_cols = [emulate.oriented_entries(c.n, g.row_offsets, g.col_indices, lo, hi)
                         for lo, hi in parts]
            f1 = np.min([emulate.first_parents(c.n, g.row_offsets, g.col_indices, lo, hi)
                         for lo, hi in parts], axis=0)
            F, G = f1.copy(), f1[f1]
            snaps = [F.copy()]
            gfc = [int(np.count_nonzero(G != np.arange(c.n)))]
            while gfc[-1]:
                Ns = []
                for rows, cols in rows_cols:
                    N = G.copy()
                    emulate.hook(rows, cols, F, G, N)
                    Ns.append(N)
                N = np.min(Ns, axis=0)
                G2 = N[N]
                gfc.append(int(np.count_nonzero(G2 != G)))
                F, G = N, G2
                snaps.append(F.copy())
            assert len(snaps) == c.iterations, (c.name, P)
            assert np.array_equal(np.stack(snaps), c.snapshots), (c.name, P)


def test_deferred_stochastic_hooks_equal_inline_hooks():
    """The dense sweep's aggressive-only hooks followed by the vertex pass's
    deferred stochastic hooks (one per lowered vertex, every value read before
    any lands) give the same f_{k+1} as hooking both targets per contribution,
    in every iteration of every golden graph, also when the sweep is split over
    ranks and merged by an elementwise min first."""
    for c in load_suite()[::3]:
        g = fb.build_csr(c.n, c.edges)
        for P in (1, 3):
            parts = [(c.n * r // P, c.n * (r + 1) // P) for r in range(P)]
            rows_cols = [emulate.oriented_entries(c.n, g.row_offsets, g.col_indices, lo, hi)
                         for lo, hi in parts]
            f1 = np.min([emulate.first_parents(c.n, g.row_offsets, g.col_indices, lo, hi)
                         for lo, hi in parts], axis=0)
            F, G = f1.copy(), f1[f1]
            k = 1
            while np.any(G != (np.arange(c.n) if k == 1 else Gprev)):
                inline, deferred = [], []
                for rows, cols in rows_cols:
                    a, b = G.copy(), G.copy()
                    emulate.hook(rows, cols, F, G, a, stochastic=True)
                    emulate.hook(rows, cols, F, G, b, stochastic=False)
                    inline.append(a)
                    deferred.append(b)
                Na, Nb = np.min(inline, axis=0), np.min(deferred, axis=0)
                emulate.deferred_stochastic(F, G, Nb)
                assert np.array_equal(Na, Nb), (c.name, P, k)
                assert np.array_equal(Na, c.snapshots[k]), (c.name, P, k)
                Gprev, F, G = G, Na, Na[Na]
                k += 1
            assert k == c.iterations, (c.name, P)
