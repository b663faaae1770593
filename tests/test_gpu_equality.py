"""GPU: the 2-PBS ASCII equality on all 128 x 128 character pairs
(reference acceptance criterion 5, tests/acceptance/main.cpp:188-217:
eq_ascii is 9*[a == b] with exactly 2 bootstraps per pair) and the
16 x 16 grid bootstrap count (criterion 6, test_kernel.cpp:473-483: 768)."""
import numpy as np
import pytest

import paper_2508_14568_b200 as L

pytestmark = pytest.mark.gpu


def test_eq_ascii_all_128x128_pairs(ctx):
    codes = np.arange(128)
    lo = ctx.encrypt(codes & 15)  # symbol 0 of every character
    hi = ctx.encrypt(codes >> 4)  # symbol 1
    a, b = np.meshgrid(codes, codes, indexing="ij")
    a, b = a.ravel(), b.ravel()
    before = ctx.stats()["pbs_count"]
    # eq_folded (equality.cpp:22-27, 59-70): eq1 = PBS(x1 - y1, eq_lut(1));
    # z = 2 (x2 - y2) + (1 - eq1); eq9 = PBS(z, eq_lut(9))
    d1 = ctx.sub(lo[a], lo[b])
    eq1 = ctx.pbs(d1, L.eq_lut(1))
    d2 = ctx.sub(hi[a], hi[b])
    z = ctx.add(ctx.scalar_mul(d2, 2), ctx.scalar_add(ctx.scalar_mul(eq1, -1), 1))
    eq9 = ctx.pbs(z, L.eq_lut(9))
    assert ctx.stats()["pbs_count"] - before == 2 * a.size
    got = ctx.decrypt(eq9)
    assert np.array_equal(got, np.where(a == b, 9, 0))
    for h in (d1, eq1, d2, z, eq9, lo, hi):
        ctx.release(h)


def test_16x16_grid_bootstraps(ctx):
    rng = np.random.default_rng(16)
    a = "".join(chr(32 + int(c)) for c in rng.integers(0, 95, 16))
    b = "".join(chr(32 + int(c)) for c in rng.integers(0, 95, 16))
    r = L.compute(a, b, ctx=ctx)
    assert r["pbs_total"] == 768 and r["pbs_equality"] == 512 and r["pbs_kernel"] == 256
    assert r["distance"] == L.wf_distance(a, b) % 32
