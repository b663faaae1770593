"""GPU: phase-noise parity of the blind rotation.

North-star criterion: where the polynomial products are not exact integer
arithmetic (here: an f64 FFT), the phase-noise variance must stay close to
an exact computation's. The oracle's mode 1 multiplies in Z_2^64[X]/(X^N+1)
exactly (schoolbook); the GPU (= oracle mode 0, bit-identical) uses the f64
FFT with a double-double BSK spectrum.

Two measurements:
  * a direct noise estimate (GPU vs exact-product blind rotations). Its
    run-to-run spread is large (the 2048 coefficients of one rotation are
    not independent samples; per-rotation std varies by ~0.1-0.2 in log2),
    so it only guards the gross level;
  * the deterministic accounting: the oracle repeats one FFT-mode rotation
    computing every external product both ways on the same input and sums
    the phase variance of the difference — the exact amount the FFT adds.
"""
import numpy as np
import pytest

import paper_2508_14568_b200 as L

pytestmark = pytest.mark.gpu


def glwe_phase(acc, S, N):
    """B - A*S (negacyclic, binary S) for a (k=1) GLWE [A | B]."""
    A, B = acc[:N].astype(np.uint64), acc[N:].astype(np.uint64)
    AS = np.zeros(N, np.uint64)
    for t in np.nonzero(S)[0]:
        rolled = np.roll(A, t)
        rolled[:t] = (np.uint64(0) - rolled[:t])
        AS += rolled
    return B - AS


def rotate(tp, e, N):
    """X^e * tp (negacyclic), e in [0, 2N)."""
    out = np.zeros(N, np.uint64)
    for j in range(N):
        s = (j - e) % (2 * N)
        out[j] = tp[s] if s < N else np.uint64((-int(tp[s - N])) % (1 << 64))
    return out


# Exact-product phase noise of one blind rotation at these parameters
# (DESIGN.md §2): BSK noise 2*N*E[d^2]*var(TUniform(2^17)) + decomposition
# rounding (1 + N/2)*2^80/3 for half the key bits, times n = 880 CMUXes.
def exact_model_var(n=880, N=2048):
    bsk = 2 * N * (2.0 ** 44 / 3) * (2.0 ** 34 / 3)
    rnd = 0.5 * (1 + N / 2) * (2.0 ** 80 / 3)
    return n * (bsk + rnd)


def test_noise_estimate_gross_level(ctx, orc):
    N, n = orc.N, orc.n
    lut = np.array(L.identity_lut(), np.int32)
    lid = ctx.lut(lut)
    tp = orc.test_poly(lut)
    rows = [orc.encrypt(v, 7000 + v) for v in (2, 5, 9, 13, 1, 6, 10, 14)]
    ms = np.stack([orc.modswitch(orc.keyswitch(r)) for r in rows])
    _, gpu = ctx.debug_blind_rotate(ms, [lid] * len(rows), glwe=True)
    fft = orc.blind_rotate_batch(ms, tp, mode=0)
    assert np.array_equal(gpu, fft)  # GPU == FFT-spec oracle, bit for bit
    exact = orc.blind_rotate_batch(ms, tp, mode=1, threads=len(rows))
    S = orc.sk_glwe()
    s_small = orc.sk_small().astype(np.int64)
    noise = {"gpu": [], "exact": []}
    for i in range(len(rows)):
        e = (-int(ms[i][n]) + int((ms[i][:n].astype(np.int64) * s_small).sum())) % (2 * N)
        want = rotate(tp, e, N)
        for name, acc in (("gpu", gpu[i]), ("exact", exact[i])):
            d = (glwe_phase(acc, S, N) - want).view(np.int64).astype(np.float64)
            noise[name].append(d)
    vg = np.var(np.concatenate(noise["gpu"]))
    ve = np.var(np.concatenate(noise["exact"]))
    # exact-product noise matches the analytical model (within the spread)
    assert 0.7 < ve / exact_model_var() < 1.4, np.log2(ve) / 2
    # 8-rotation estimate of the ratio: expected ~1.19 (accounting test
    # below), observed spread of such estimates ~+-0.25
    assert 1 / 1.1 <= vg / ve <= 1.6, (vg / ve, np.log2(vg) / 2, np.log2(ve) / 2)


def test_fft_added_phase_variance(orc):
    lut = np.array(L.identity_lut(), np.int32)
    tp = orc.test_poly(lut)
    vs = []
    for v in (3, 11):
        ms = orc.modswitch(orc.keyswitch(orc.encrypt(v, 7100 + v)))
        vs.append(orc.fft_phase_error_var(ms, tp))
    frac = float(np.mean(vs)) / exact_model_var()
    # Measured 2^95.54 per rotation = 0.19 of the exact-product noise
    # (2^97.9): the f64 rounding of the digit spectrum and of the inverse
    # transform, each ~half. A plain-f64 BSK spectrum (TFHE-rs's way) adds
    # 2^96.19 = 0.31; the double-double BSK removes that third of the error.
    assert 0.12 < frac < 0.25, (frac, np.log2(vs))


@pytest.mark.parametrize("pair_max", [0, 1 << 30])
def test_exact_mask_product_mode(pair_max, monkeypatch):
    """lv_params.exact_mask_product = 1: bit-exact with the oracle's split
    (H 2^43 + Lo) mask product — through the single-CTA exact kernel
    (pair_max 0) and the CTA-pair exact kernel — decrypts correctly, and the
    FFT's added phase variance drops to a negligible fraction of the exact
    noise."""
    monkeypatch.setenv("LVB_BR_PAIR_MAX", str(pair_max))
    from oracle.oracle import Oracle, default_params as oracle_params
    op = oracle_params()
    op.exact_mask_product = 1
    orc = Oracle(seed=0, params=op)
    p = L.default_params()
    p.exact_mask_product = 1
    c = L.Context(seed=0, params=p)
    try:
        lut = np.array(L.eq_lut(9), np.int32)
        lid = c.lut(lut)
        tp = orc.test_poly(lut)
        rows = [orc.encrypt(v, 9300 + v) for v in (0, 7, 15)]
        ms = np.stack([orc.modswitch(orc.keyswitch(r)) for r in rows])
        _, glwe = c.debug_blind_rotate(ms, [lid] * len(rows), glwe=True)
        assert np.array_equal(glwe, orc.blind_rotate_batch(ms, tp, mode=0))
        vals = [3, 0, 12, 0, 31 - 16]
        out = c.pbs(c.encrypt(vals), lut)
        assert list(c.decrypt(out)) == [L.negacyclic_eval(lut, v) for v in vals]
        r = L.compute("monday", "friday", ctx=c)
        assert r["distance"] == 3 and r["pbs_total"] == 108
        frac = orc.fft_phase_error_var(ms[1], orc.test_poly(np.array(L.identity_lut(), np.int32)))
        frac /= exact_model_var()
        assert frac < 0.005, frac  # measured 2^85.8 / 2^97.9 = 2.3e-4
    finally:
        c.close()


@pytest.mark.parametrize("exact_mask", [0, 1])
def test_measured_output_noise_4096(exact_mask):
    """North-star noise criterion, measured: the output phase error of 4096
    independent bootstraps against the exact-product model. Default keys:
    1 + 0.19 predicted (0.91x the reference's f64-spectrum algorithm);
    exact-mask keys: 1.0002 predicted. Sampling std error ~2.5%."""
    p = L.default_params()
    p.exact_mask_product = exact_mask
    c = L.Context(seed=11, params=p)
    try:
        vals = [(5 * i + 3) % 16 for i in range(4096)]
        out = c.pbs(c.encrypt(vals), L.identity_lut())
        e = (c.phase(out) - np.asarray(vals, np.uint64) * np.uint64(1 << 59)).view(np.int64)
        ratio = float(np.var(e.astype(np.float64))) / exact_model_var()
        lo, hi = (1.07, 1.32) if exact_mask == 0 else (0.89, 1.11)
        assert lo < ratio < hi, ratio
    finally:
        c.close()


def _phase_errors(mode: int, vals):
    p = L.default_params()
    p.exact_mask_product = mode
    c = L.Context(seed=11, params=p)
    try:
        out = c.pbs(c.encrypt(vals), L.identity_lut())
        return (c.phase(out) - np.asarray(vals, np.uint64) * np.uint64(1 << 59)).view(np.int64)
    finally:
        c.close()


def test_noise_vs_reference_algorithm_measured():
    """North-star noise criterion against a MEASURED denominator: the same
    4096 bootstraps (same seed, so the same keys, encryptions and exact-
    product noise) with the reference's algorithm — exact_mask_product = 2,
    the TFHE-rs f64-FFT PBS whose BSK spectrum is the plain f64 transform —
    on this GPU. The shared exact-product noise cancels in the ratio, so
    4096 samples pin it to about +-1%. Ours (double-double BSK spectrum)
    and the exact-mask keys must stay within 1.1x of it; measured r02:
    0.91x and 0.76x."""
    vals = [(5 * i + 3) % 16 for i in range(4096)]
    ref = float(np.var(_phase_errors(2, vals).astype(np.float64)))
    assert 1.15 < ref / exact_model_var() < 1.55, ref / exact_model_var()  # model 1 + 0.31
    for mode, hi in ((0, 1.0), (1, 0.85)):
        v = float(np.var(_phase_errors(mode, vals).astype(np.float64)))
        assert v / ref < hi < 1.1, (mode, v / ref)
