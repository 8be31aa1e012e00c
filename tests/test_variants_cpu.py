"""The device schedule of the hooking variants (init forms, filters, two-commit
shortcut), restated in numpy, reproduces the reference's own traces of every
HookingConfig and simplified_sv (tests/golden/variants.npz, made by
tests/golden/make_variant_golden.py from svcc itself)."""

import paper_1910_05971_b200 as fb
import emulate_variants
from golden_io import load_variants, variant_graphs
from paper_1910_05971_b200 import generators as gen


def test_variant_schedule_matches_reference_traces():
    runs, extra = load_variants()
    graphs = variant_graphs()
    for name, digest in extra.items():
        assert gen.pairs_digest(graphs[name][1]) == digest, name
    csr = {}
    for name, code, iters, gfc, fc, digest in runs:
        if name.startswith("x:config1"):
            continue                       # the largest; covered on the GPU
        if name not in csr:
            n, e = graphs[name]
            csr[name] = (n, fb.build_csr(n, e))
        n, g = csr[name]
        got = emulate_variants.run(n, g.row_offsets, g.col_indices, code)
        assert got == (iters, gfc, fc, digest), (name, code)
