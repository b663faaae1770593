"""GPU end to end: decrypted distances and every counter of
cli::compute_report equal the reference's (tests/golden, produced by the
reference's own SimBackend), through the wavefront scheduler."""
import pytest

import paper_2508_14568_b200 as L
from paper_2508_14568_b200 import workloads as W

pytestmark = pytest.mark.gpu

ERR = {"BandTooNarrow": L.BandTooNarrow, "CharNotInAlphabet": L.CharNotInAlphabet,
       "InvalidParams": L.InvalidParams, "CharNotInSubset": L.CharNotInSubset}

FIELDS = ["distance", "visited_cells", "pbs_total", "pbs_equality", "pbs_kernel", "refresh_count",
          "preprocessing_pbs", "max_key_variance", "linear_ops", "half_width"]


def run_case(case):
    return L.compute(case["a"], case["b"], mode=case["mode"],
                     ell=case["ell"] if case["mode"] == "approx" else None,
                     encoding=case["encoding"], budget=case["budget"],
                     key_encoding=case["key_encoding"], preprocess=case["preprocess"])


def test_reference_cases(golden):
    for case in golden["cases"]:
        if "error" in case:
            with pytest.raises(ERR[case["error"]]):
                run_case(case)
            continue
        got = run_case(case)
        want = case["report"]
        for f in FIELDS:
            assert got[f] == want[f], (case["a"], case["b"], f, got[f], want[f])


def test_worked_examples():
    r = L.compute("monday", "friday")  # test_kernel.cpp:230-249
    assert (r["distance"], r["pbs_kernel"], r["pbs_equality"], r["refresh_count"]) == (3, 36, 72, 0)
    assert L.compute("KID", "SIT")["distance"] == 2
    assert L.compute("zzzz", "zzzz", mode="skip")["distance"] == 0


def test_config1(golden):
    a, b = W.cfg1()
    got = L.compute(a, b)
    for f in FIELDS:
        assert got[f] == golden["configs"]["cfg1"]["report"][f], f


def test_config3(golden):
    a, b = W.cfg3()
    got = L.compute(a, b)
    for f in FIELDS:
        assert got[f] == golden["configs"]["cfg3"]["report"][f], f


def test_config4_preprocessed(golden):
    a, b = W.cfg4()
    got = L.compute(a, b, encoding="dna4", preprocess=True)
    for f in FIELDS:
        assert got[f] == golden["configs"]["cfg4"]["report"][f], f


def test_config5_full_batch(golden):
    """BASELINE configs[4] in full: all 256 pairs (128 x 128 printable ASCII,
    15% edits) in one compute_batch() wavefront (cli.cpp:164-210 batch mode,
    acceptance criterion 11). Every pair's decrypted distance and every
    RunReport counter equal the compiled reference's (golden cfg5). ~4 min."""
    pairs = W.cfg5(256)
    reps = L.compute_batch(pairs)
    assert len(reps) == 256
    for i, (rep, want) in enumerate(zip(reps, golden["configs"]["cfg5"])):
        assert (want["a"], want["b"]) == pairs[i]
        for f in FIELDS:
            if f in rep:  # compute_batch reports carry every counter but preprocessing_pbs
                assert rep[f] == want["report"][f], (i, f, rep[f], want["report"][f])
    assert sum(r["distance"] for r in reps) == 4557


def test_empty_operands():
    assert L.compute("", "")["distance"] == 0
    assert L.compute("abc", "")["distance"] == 3
    assert L.compute("", "abcd")["distance"] == 4
    with pytest.raises(L.BandTooNarrow):
        L.compute("ab", "", mode="skip")


def test_long_pairs(golden):
    """Long single pairs from the compiled reference (golden "long"): a
    300 x 300 printable pair whose keys reach the default budget (40
    refreshes; waves grow past the CTA-pair range onto the throughput
    kernel) and a 256 x 256 skip-band DNA pair. Every RunReport counter and
    the distance equal the reference's."""
    for case in golden["long"]:
        rep = L.compute(case["a"], case["b"], mode=case["mode"], encoding=case["encoding"])
        want = case["report"]
        for f in ("distance", "half_width", "visited_cells", "pbs_total", "pbs_equality",
                  "pbs_kernel", "refresh_count", "max_key_variance", "linear_ops"):
            assert rep[f] == want[f], (f, rep[f], want[f])


def test_eq9_provider_traversal():
    """kernel::distance with a caller-supplied Eq9Provider (kernel.hpp:162-199,
    lv_edit_distance_eq9): encrypted 9*[a_i == b_j] handles from the caller,
    asked once per in-band cell; the distance and the counters match the
    encrypted-vs-encrypted traversal's kernel part (no equality bootstraps)."""
    from paper_2508_14568_b200 import leuven as LV
    ctx = L.Context(seed=21)
    a, b = "kitten", "sitting"
    asked = []

    def provider(i, j):
        asked.append((i, j))
        return int(ctx.encrypt([9 if a[i - 1] == b[j - 1] else 0])[0])
    run = LV.distance(ctx, provider, len(a), len(b), LV.BandSpec.exact(len(a), len(b)))
    assert int(ctx.decrypt([run.score])[0]) == 3
    assert len(asked) == len(set(asked)) == 42
    assert (run.kernel_pbs, run.equality_pbs, run.visited_cells) == (42, 0, 42)
    band = LV.BandSpec.skip(len(a), len(b))
    asked.clear()
    run = LV.distance(ctx, provider, len(a), len(b), band)
    assert int(ctx.decrypt([run.score])[0]) == LV.banded_distance(a, b, band.half_width) % 32
    assert len(asked) == run.visited_cells < 42
    ctx.close()
