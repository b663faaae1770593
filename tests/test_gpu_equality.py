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


@pytest.mark.parametrize("encoding", ["negated", "original"])
def test_cell_all_18_inputs(ctx, golden, encoding):
    """test_kernel.cpp:101-142: the cell over all 18 inputs (dv, dh in
    {-1, 0, 1}, eq in {0, 1}) in both key encodings, one bootstrap each:
    key = 3 dh - dv + 9 eq + 4 (negated) or dv + 3 dh + 9 eq + 4 (original,
    kernel.cpp:152-163), step = PBS(key, min-LUT) = 1 + min(-eq, dv, dh),
    dv' = step - dh, dh' = step - dv — built here from encrypted operands
    with the public linear ops."""
    lut = golden["luts"]["minlut-" + encoding]
    lid = ctx.lut(lut)
    combos = [(dv, dh, eq) for dv in (-1, 0, 1) for dh in (-1, 0, 1) for eq in (0, 1)]
    dv = ctx.encrypt([v % 32 for v, _, _ in combos])
    dh = ctx.encrypt([h % 32 for _, h, _ in combos])
    eq9 = ctx.encrypt([9 * e for _, _, e in combos])
    if encoding == "negated":
        key = ctx.sub(ctx.scalar_mul(dh, [3] * 18), dv)
    else:
        key = ctx.add(dv, ctx.scalar_mul(dh, [3] * 18))
    key = ctx.scalar_add(ctx.add(key, eq9), [4] * 18)
    before = ctx.stats()["pbs_count"]
    step = ctx.pbs(key, lut_ids=[lid] * 18)
    assert ctx.stats()["pbs_count"] - before == 18  # exactly one bootstrap per cell
    want = [(1 + min(-e, v, h)) % 32 for v, h, e in combos]
    assert list(ctx.decrypt(step)) == want
    assert list(ctx.decrypt(ctx.sub(step, dh))) == [(w - h) % 32 for w, (_, h, _) in zip(want, combos)]
    assert list(ctx.decrypt(ctx.sub(step, dv))) == [(w - v) % 32 for w, (v, _, _) in zip(want, combos)]


def test_equality_inputs_checked_against_budget(ctx):
    """eq4 / fold_step go through SimBackend::pbs in the
    reference (equality.cpp:22-70), which throws NoiseBudgetExceeded on an
    over-noisy input. Symbols scaled by scalar_mul(64) (variance 4096 >
    4000) must be rejected before anything is launched, in the traversal
    and in the preprocessing table build; fresh symbols pass."""
    spec = L.AlphabetSpec.ascii7()
    xa = L.encrypt_string("ab", spec, ctx)
    xb = L.encrypt_string("ac", spec, ctx)
    bad = L.EncryptedString(ctx.scalar_mul(xa.chars.reshape(-1), 64).reshape(xa.chars.shape))
    band = L.BandSpec.exact(2, 2)
    with pytest.raises(L.NoiseBudgetExceeded):
        L.distance_encrypted(ctx, bad, xb, band)
    with pytest.raises(L.NoiseBudgetExceeded):
        L.build_eq_table(ctx, bad, spec)
    run = L.distance_encrypted(ctx, xa, xb, band)
    assert int(ctx.decrypt([run.score])[0]) == 1
