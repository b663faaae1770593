"""GPU: banded traversal contracts (reference acceptance criteria 6 and 10,
tests/acceptance/main.cpp:221-265 and 464-503): banded bootstrap counts
follow the closed form, and approx(ell) is exact when the distance is
below ell and never below the true distance otherwise."""
import numpy as np
import pytest

import paper_2508_14568_b200 as L

pytestmark = pytest.mark.gpu


def _rand(rng, n):
    return "".join(chr(32 + int(c)) for c in rng.integers(0, 95, n))


def _mutate(rng, s, edits):
    s = list(s)
    for _ in range(edits):
        if not s:
            break
        op, pos = int(rng.integers(0, 3)), int(rng.integers(0, len(s)))
        if op == 0:
            s[pos] = chr(32 + int(rng.integers(0, 95)))
        elif op == 1:
            del s[pos]
        else:
            s.insert(pos, chr(32 + int(rng.integers(0, 95))))
    return "".join(s)


def test_banded_bootstrap_counts(ctx):
    rng = np.random.default_rng(106)
    a, b = _rand(rng, 16), _rand(rng, 16)
    r = L.compute(a, b, mode="skip", ctx=ctx)
    assert r["half_width"] == 8 and r["pbs_kernel"] == L.band_cell_count(16, 8)
    a, b = _rand(rng, 100), _rand(rng, 100)
    r = L.compute(a, b, mode="approx", ell=10, ctx=ctx)
    assert r["pbs_kernel"] == 1990 and r["visited_cells"] == 1990


def test_approximation_contract(ctx):
    rng = np.random.default_rng(110)
    spec = L.AlphabetSpec.ascii7()
    pairs = []
    for t in range(120):
        m = 2 + int(rng.integers(0, 13))
        a = _rand(rng, m)
        b = _rand(rng, m) if t % 3 == 0 else _mutate(rng, a, int(rng.integers(0, 6)))
        while len(b) + 2 < len(a):
            b += "x"
        while len(a) + 2 < len(b):
            b = b[:-1]
        pairs.append((a, b))
    enc = [(L.encrypt_string(a, spec, ctx), L.encrypt_string(b, spec, ctx)) for a, b in pairs]
    checked = at_ell = exact_at_ell = 0
    for ell in (2, 4, 8):
        runs = L.distance_batch(ctx, enc, [L.BandSpec.approx(ell)] * len(pairs))
        got = ctx.decrypt([r.score for r in runs])
        ctx.release([r.score for r in runs])
        for (a, b), g in zip(pairs, got):
            want = L.wf_distance(a, b)
            checked += 1
            if want <= ell - 1:
                assert g == want, (a, b, ell, g, want)
            else:
                assert g >= want, (a, b, ell, g, want)  # distances < 32: no wrap
            if want == ell:
                at_ell += 1
                exact_at_ell += g == want
    assert checked == 360
