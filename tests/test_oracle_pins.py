"""CPU: pins the oracle (test infrastructure) against the reference's golden
vectors and against itself (FFT-spec mode vs exact-integer mode)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2508_14568_b200 import workloads as W


@pytest.fixture(scope="module")
def toy():
    return O.Oracle(7, O.toy_params())


def test_philox_known_answer():
    # Random123 Philox4x32-10 KAT: ctr=0, key=0 -> 6627e8d5 e169c58d bc57ac4c 9b00dbd8
    out = (O.ctypes.c_uint32 * 4)()
    O.lib().orc_philox(0, 0, 0, out)
    assert list(out) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


def test_tuniform_range_and_moments():
    vals = np.array([O.lib().orc_tuniform(3, 9, i, 4) for i in range(20000)])
    assert vals.min() == -16 and vals.max() == 16
    # TUniform(b) variance = (2^(2b+1) + 1) / 6
    assert abs(vals.var() - (2 ** 9 + 1) / 6) < 5


def test_luts_match_reference_tables(golden):
    luts = golden["luts"]
    assert luts["minlut-original"] == [0, 0, 0, 0, 1, 1, 0, 1, 1, 0, 0, 0, 0, 0, 0, 0]
    assert luts["eqlut9"] == [9] + [0] * 15
    assert luts["identity"] == list(range(16))


@pytest.mark.parametrize("name", ["minlut-original", "minlut-negated", "eqlut1", "eqlut9", "identity"])
def test_pbs_realises_negacyclic_eval(toy, golden, name):
    """decrypt(PBS(enc(x), lut)) == negacyclic_eval(lut, x) (lut.cpp:9-16), all 32 x."""
    lut = np.array(golden["luts"][name], np.int32)
    cts = np.stack([toy.encrypt(x, 100 + x) for x in range(32)])
    outs = toy.pbs_batch(cts, np.tile(lut, (32, 1)))
    got = [toy.decrypt(o) for o in outs]
    assert got == [O.negacyclic_eval(lut, x) for x in range(32)]


def test_exact_and_fft_modes_agree_on_values(toy):
    lut = np.array([(5 * i + 1) % 32 for i in range(16)], np.int32)
    for x in (0, 7, 15, 16, 31):
        c = toy.encrypt(x, 500 + x)
        a, b = toy.pbs(c, lut, 0), toy.pbs(c, lut, 1)
        assert toy.decrypt(a) == toy.decrypt(b) == O.negacyclic_eval(lut, x)


def test_fft_roundtrip_is_exact_for_small_polys(toy):
    rng = np.random.default_rng(3)
    p = rng.integers(-2 ** 22, 2 ** 22, toy.N)
    assert np.array_equal(toy.fft_backward(toy.fft_forward(p)).view(np.int64), p)


def test_keyswitch_preserves_phase(toy):
    c = toy.encrypt(13, 77)
    s = toy.keyswitch(c)
    d = (toy.phase_small(s) - toy.phase(c)) % 2 ** 64
    d = d - 2 ** 64 if d >= 2 ** 63 else d
    assert abs(d) < 2 ** 56  # well inside half a plaintext step (2^58)


def test_workload_generator_matches_reference_runs(golden):
    cfg = golden["configs"]
    a, b = W.cfg1()
    assert (cfg["cfg1"]["a"], cfg["cfg1"]["b"]) == (a, b)
    assert cfg["cfg1"]["report"]["distance"] == W.wf_distance(a, b) == 7
    a, b = W.cfg3()
    assert cfg["cfg3"]["report"]["distance"] == 31 and (cfg["cfg3"]["a"], cfg["cfg3"]["b"]) == (a, b)
    a, b = W.cfg4()
    assert cfg["cfg4"]["report"]["distance"] == 6 and len(b) == 62
    assert cfg["cfg4"]["report"]["preprocessing_pbs"] == 256
    h = 0
    for m in W.cfg2():
        h = (h * 31 + m) & 0xFFFFFFFF
    assert h == cfg["cfg2"]["message_hash"] == 1181287816
    assert cfg["cfg2"]["outputs"] == W.cfg2()  # identity LUT on [0,16)
    pairs = W.cfg5()
    assert [p["a"] for p in cfg["cfg5"]] == [a for a, _ in pairs]
    assert sum(p["report"]["distance"] for p in cfg["cfg5"]) == 4557
    assert sum(p["report"]["pbs_total"] for p in cfg["cfg5"]) == 12578688


def test_golden_distances_equal_wagner_fischer(golden):
    for c in golden["cases"]:
        if "error" in c or c["mode"] != "exact":
            continue
        assert c["report"]["distance"] == W.wf_distance(c["a"], c["b"]) % 32


def _has_avx512():
    try:
        flags = set(open("/proc/cpuinfo").read().split())
    except OSError:
        return False
    return {"avx512f", "avx512dq", "avx512bw", "avx512vl", "fma"} <= flags


@pytest.mark.skipif(not _has_avx512(), reason="the CPU-baseline build needs AVX-512")
def test_cpu_baseline_build_bit_identical():
    """The CPU baseline (the -O3 x86-64-v4 oracle build, 8 ciphertexts per
    AVX-512 lane set) equals the scalar checker bit for bit, on a ragged
    batch (11 = 8 + 3 lanes) with two LUTs."""
    import numpy as np
    from oracle import oracle as O
    slow, fast = O.Oracle(0), O.Oracle(0, fast=True)
    rows = np.stack([slow.encrypt(v % 32, 500 + v) for v in range(11)])
    luts = np.tile(np.arange(16, dtype=np.int32), (11, 1))
    luts[1::2] = np.array([(3 * x + 1) % 16 for x in range(16)], np.int32)
    want = slow.pbs_batch(rows, luts)
    assert np.array_equal(fast.pbs_batch(rows, luts), want)
    assert np.array_equal(fast.pbs_batch_simd(rows, luts), want)
