"""GPU parity of the PBS path against the CPU oracle, stage by stage, at the
default (production) parameter set. Integer stages and the f64 FFT
external product are required to be BIT-EXACT (the FFT operation order is
specified in oracle/tfhe_oracle.c and reproduced by csrc/fft.cuh)."""
import numpy as np
import pytest

import paper_2508_14568_b200 as L
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_keygen_bit_exact(ctx, orc):
    sks, skg, ksk, bskf = ctx.debug_keys()
    assert np.array_equal(sks, orc.sk_small())
    assert np.array_equal(skg, orc.sk_glwe())
    assert np.array_equal(ksk, orc.ksk())
    assert np.array_equal(bskf.view(np.uint64), orc.bskf().view(np.uint64))


def test_fft_bit_exact(ctx, orc):
    rng = np.random.default_rng(11)
    for scale in (2 ** 22, 2 ** 62):
        p = rng.integers(-scale, scale, 2048)
        spec, rt = ctx.debug_fft(p)
        want = orc.fft_forward(p)
        assert np.array_equal(spec.view(np.uint64), want.view(np.uint64))
        assert np.array_equal(rt, orc.fft_backward(want))


def test_encrypt_bit_exact_and_decrypts(golden):
    c = L.Context(seed=0)
    vals = list(range(32)) * 2
    h = c.encrypt(vals)
    rows = c.export(h)
    o = O.Oracle(0)
    for i, v in enumerate(vals):
        assert np.array_equal(rows[i], o.encrypt(v, i))
    assert list(c.decrypt(h)) == vals
    c.close()


def test_keyswitch_bit_exact(ctx, orc):
    rows = np.stack([orc.encrypt(v, 1000 + v) for v in range(24)])
    got = ctx.debug_keyswitch(rows)
    for i in range(len(rows)):
        assert np.array_equal(got[i], orc.keyswitch(rows[i]))


def test_blind_rotate_bit_exact(ctx, orc, golden):
    lut = np.array(golden["luts"]["minlut-negated"], np.int32)
    lid = ctx.lut(lut)
    rows = [orc.encrypt(v, 2000 + v) for v in range(6)]
    ms = np.stack([orc.modswitch(orc.keyswitch(r)) for r in rows])
    got = ctx.debug_blind_rotate(ms, [lid] * len(rows))
    tp = orc.test_poly(lut)
    for i in range(len(rows)):
        want = orc.sample_extract(orc.blind_rotate(ms[i], tp))
        assert np.array_equal(got[i], want)


def test_pbs_bit_exact_all_luts(ctx, orc, golden):
    names = ["identity", "minlut-negated", "minlut-original", "eqlut1", "eqlut9"]
    luts = np.array([golden["luts"][n] for n in names], np.int32)
    ids = np.array([ctx.lut(l) for l in luts], np.uint32)
    xs = np.arange(40) % 32
    rows = np.stack([orc.encrypt(int(x), 3000 + i) for i, x in enumerate(xs)])
    which = np.arange(40) % len(names)
    got = ctx.pbs_host(rows, ids[which])
    want = orc.pbs_batch(rows, luts[which])
    assert np.array_equal(got, want)
    for i, x in enumerate(xs):
        assert orc.decrypt(got[i]) == L.negacyclic_eval(luts[which[i]], int(x))


def test_pbs_host_equals_device_path(ctx, golden):
    # 2000 items (several blind-rotation waves, mixed LUTs): the host-buffer
    # entry point must equal the handle path bit for bit, in order
    luts = [golden["luts"][n] for n in ("identity", "minlut-negated", "eqlut9")]
    ids = np.array([ctx.lut(l) for l in luts], np.uint32)
    vals = [(7 * i) % 16 for i in range(2000)]
    cts = ctx.encrypt(vals)
    rows = ctx.export(cts)
    which = ids[np.arange(2000) % 3]
    got = ctx.pbs_host(rows, which)
    dev = ctx.pbs(cts, lut_ids=which)
    assert np.array_equal(got, ctx.export(dev))
    ctx.release(cts)
    ctx.release(dev)


def test_pbs_handles_budget_and_counters(golden):
    c = L.Context(seed=5, budget=25.0)  # NoiseParams::tight(), backend.hpp:29
    lut = [(x - 4 + 16) % 16 for x in range(16)]  # test_backend.cpp:16-24
    out = c.pbs(c.encrypt([5]), lut)
    assert list(c.decrypt(out)) == [1]
    assert list(c.variance(out)) == [1]
    assert c.stats()["pbs_count"] == 1
    noisy = c.trivial([0])
    for _ in range(25):
        noisy = c.add(noisy, c.encrypt([0]))
    assert list(c.variance(noisy)) == [25]
    c.pbs(noisy, lut)
    noisy = c.add(noisy, c.encrypt([0]))
    with pytest.raises(L.NoiseBudgetExceeded):
        c.pbs(noisy, lut)
    seven = c.refresh(c.encrypt([7]))
    assert list(c.decrypt(seven)) == [7]
    with pytest.raises(L.ValueOutsideLutHalf):
        c.refresh(c.encrypt([16]))
    assert c.stats()["refresh_count"] == 1
    with pytest.raises(L.OutOfRangeValue):
        c.encrypt([32])
    c.close()


def test_linear_ops_follow_reference(ctx):
    a = ctx.encrypt([3])
    assert list(ctx.decrypt(ctx.scalar_mul(a, 3))) == [9]
    assert list(ctx.variance(ctx.scalar_mul(a, 3))) == [9]
    gone = ctx.sub(a, a)
    assert list(ctx.decrypt(gone)) == [0] and list(ctx.variance(gone)) == [0]
    assert list(ctx.decrypt(ctx.scalar_add(ctx.encrypt([30]), 5))) == [3]
    assert list(ctx.decrypt(ctx.scalar_mul(ctx.encrypt([1]), -1))) == [31]
    x, y = ctx.encrypt([1]), ctx.encrypt([2])
    shared = ctx.sub(x, y)
    assert ctx.predict_variance([(x[0], 1), (y[0], 3)]) == 10
    assert ctx.predict_variance([(x[0], 1), (shared[0], 1)]) == 5


def test_random_linear_circuits(ctx):
    rng = np.random.default_rng(11)  # test_backend.cpp:67-110
    for _ in range(20):
        plain = list(rng.integers(0, 32, 4))
        cts = list(ctx.encrypt(plain))
        for _ in range(12):
            i, j = rng.integers(0, len(cts), 2)
            op = rng.integers(0, 4)
            if op == 0:
                cts.append(ctx.add([cts[i]], [cts[j]])[0]); plain.append((plain[i] + plain[j]) % 32)
            elif op == 1:
                cts.append(ctx.sub([cts[i]], [cts[j]])[0]); plain.append((plain[i] - plain[j]) % 32)
            elif op == 2:
                k = int(rng.integers(0, 7)) - 3
                cts.append(ctx.scalar_mul([cts[i]], k)[0]); plain.append((plain[i] * k) % 32)
            else:
                k = int(rng.integers(0, 32))
                cts.append(ctx.scalar_add([cts[i]], k)[0]); plain.append((plain[i] + k) % 32)
        assert list(ctx.decrypt(cts)) == [int(p) for p in plain]


@pytest.mark.parametrize("pair_max", [0, 1 << 30])
def test_blind_rotate_variants_bit_exact(orc, pair_max, monkeypatch):
    """Single-CTA (pair_max 0) and CTA-pair (cluster of 2 SMs, DSMEM
    spectrum exchange) blind rotations both equal the FFT-spec oracle bit
    for bit, including the whole GLWE accumulator."""
    monkeypatch.setenv("LVB_BR_PAIR_MAX", str(pair_max))
    c = L.Context(seed=0)
    try:
        lut = np.array(L.eq_lut(9), np.int32)
        lid = c.lut(lut)
        tp = orc.test_poly(lut)
        rows = [orc.encrypt(v, 9100 + v) for v in (0, 3, 7, 12, 15)]
        ms = np.stack([orc.modswitch(orc.keyswitch(r)) for r in rows])
        out, glwe = c.debug_blind_rotate(ms, [lid] * len(rows), glwe=True)
        want = orc.blind_rotate_batch(ms, tp, mode=0)
        assert np.array_equal(glwe, want)
        for i in range(len(rows)):
            assert np.array_equal(out[i], orc.sample_extract(want[i]))
    finally:
        c.close()


def test_concurrent_host_threads_share_one_context(golden):
    """backend.hpp:79-82: concurrent operations from several host threads on
    one backend are safe and the counters add up (the context mutex
    serialises calls onto its stream; ctypes releases the GIL)."""
    import threading
    c = L.Context(seed=21)
    lut = golden["luts"]["minlut-negated"]
    lid = c.lut(lut)
    errors, results = [], {}

    def work(k):
        try:
            vals = [(k * 7 + i) % 32 for i in range(50)]
            got = []
            for _ in range(3):
                out = c.pbs(c.encrypt(vals), lid)
                got.append(list(c.decrypt(out)))
            results[k] = (vals, got)
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    try:
        assert not errors, errors
        for k, (vals, got) in results.items():
            want = [L.negacyclic_eval(lut, v) for v in vals]
            assert all(g == want for g in got), k
        assert c.stats()["pbs_count"] == 6 * 3 * 50
    finally:
        c.close()


def test_context_device_selection():
    """lv_params.device picks the context's GPU (-1: the current device);
    an index past the device count is InvalidParams."""
    c = L.Context(seed=2, device=0)
    try:
        assert list(c.decrypt(c.pbs(c.encrypt([4]), L.identity_lut()))) == [4]
    finally:
        c.close()
    with pytest.raises(L.InvalidParams):
        L.Context(seed=2, device=1 << 20)


def test_repeated_batches_bit_identical(ctx):
    """Race guard (compute-sanitizer is unavailable on the GPU pool): a
    4096-item batch on the throughput kernel and a 48-item batch on the
    CTA-pair kernel, each repeated, give bit-identical ciphertexts."""
    lid = ctx.lut(L.identity_lut())
    for n in (4096, 48):
        h = ctx.encrypt([i % 16 for i in range(n)])
        ref = ctx.export(ctx.pbs(h, lid))
        for _ in range(2):
            assert np.array_equal(ref, ctx.export(ctx.pbs(h, lid))), n
        ctx.release(h)


@pytest.mark.parametrize("pair_max", [0, 1 << 30])
def test_other_lwe_dimension_bit_exact(golden, pair_max, monkeypatch):
    """n is a runtime parameter (only N, k and the gadgets are compiled in):
    n = 630 keys, key switch and blind rotation stay bit-exact with the
    oracle at the same parameters, on both blind-rotation kernels."""
    monkeypatch.setenv("LVB_BR_PAIR_MAX", str(pair_max))
    from oracle.oracle import Oracle, default_params as oracle_params
    op = oracle_params()
    op.n = 630
    orc = Oracle(seed=3, params=op)
    p = L.default_params()
    p.n = 630
    c = L.Context(seed=3, params=p)
    try:
        lut = np.array(golden["luts"]["minlut-negated"], np.int32)
        lid = c.lut(lut)
        rows = np.stack([orc.encrypt(v, 4000 + v) for v in (1, 6, 11, 17)])
        want = orc.pbs_batch(rows, np.tile(lut, (4, 1)))
        assert np.array_equal(c.pbs_host(rows, [lid] * 4), want)
        sks, _, ksk, _ = c.debug_keys()
        assert np.array_equal(sks, orc.sk_small()) and np.array_equal(ksk, orc.ksk())
    finally:
        c.close()


def test_contexts_of_different_n_coexist(ctx, orc, golden):
    """Kernel attributes are process-wide: creating a context with a smaller
    n must not shrink the shared-memory limit that the default context's
    launches (larger n) need (regression: 'invalid argument' on the next
    n = 880 launch after an n = 630 context was created)."""
    p = L.default_params()
    p.n = 630
    small = L.Context(seed=3, params=p)
    try:
        lut = np.array(golden["luts"]["minlut-negated"], np.int32)
        rows = np.stack([orc.encrypt(v, 5000 + v) for v in (2, 9, 20)])
        want = orc.pbs_batch(rows, np.tile(lut, (3, 1)))
        assert np.array_equal(ctx.pbs_host(rows, [ctx.lut(lut)] * 3), want)
    finally:
        small.close()


def test_pbs_bit_exact_throughput_kernel(orc, golden, monkeypatch):
    # waves above br_pair_max run the one-CTA-per-item throughput kernel
    # (blind_rotate_kernel); 301 items = several CTAs per SM, a partial wave
    monkeypatch.setenv("LVB_BR_PAIR_MAX", "0")
    c = L.Context(seed=0)
    names = ["identity", "minlut-negated", "eqlut9"]
    luts = np.array([golden["luts"][n] for n in names], np.int32)
    ids = np.array([c.lut(l) for l in luts], np.uint32)
    count = 301
    xs = (np.arange(count) * 7) % 32
    rows = np.stack([orc.encrypt(int(x), 5000 + i) for i, x in enumerate(xs)])
    which = np.arange(count) % len(names)
    got = c.pbs_host(rows, ids[which])
    want = orc.pbs_batch(rows, luts[which])
    assert np.array_equal(got, want)
    c.close()


def _host_has_avx512():
    try:
        flags = set(open("/proc/cpuinfo").read().split())
    except OSError:
        return False
    return {"avx512f", "avx512dq", "avx512bw", "avx512vl", "fma"} <= flags


@pytest.mark.skipif(not _host_has_avx512(), reason="the fast oracle build needs AVX-512")
def test_cfg2_4096_ciphertexts_bit_exact(ctx):
    """The whole BASELINE configs[1] batch (4096 cfg2 messages, identity LUT,
    keys seed 0) through the product path — one throughput-kernel launch
    over 9+ waves — equals the oracle's PBS word for word on every output
    LWE (the oracle's lane-vectorised build, itself pinned bit-identical to
    the scalar checker by tests/test_oracle_pins.py)."""
    from oracle import oracle as O
    from paper_2508_14568_b200 import workloads as W
    o = O.Oracle(0, fast=True)
    vals = W.cfg2()
    rows = np.stack([o.encrypt(v, i) for i, v in enumerate(vals)])
    lid = ctx.lut(L.identity_lut())
    got = ctx.pbs_host(rows, np.full(len(vals), lid, np.uint32))
    want = o.pbs_batch_simd(rows, np.tile(np.arange(16, dtype=np.int32), (len(vals), 1)))
    assert want is not None
    same = np.all(got == want, axis=1)
    assert same.all(), f"{int((~same).sum())} of 4096 differ"
    assert [o.decrypt(r) for r in got[:64]] == vals[:64]
