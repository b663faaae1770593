"""CPU: the C-ABI library loads and exports every declared symbol; the
host-side symbolic planner (no device work) reproduces the reference's
per-cell key variances, refresh placement and counters exactly."""
import os
import re

import pytest

import paper_2508_14568_b200 as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "leuven_b200.h")).read()
    decl = r"^(?:int|void|const char\*)\s+(lv_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(decl, text, flags=re.M)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(L.EXPORTS)


def test_library_exports_every_symbol(product_lib):
    for name in declared_symbols():
        assert hasattr(product_lib, name), name
    assert product_lib.lv_abi_version() == 1


def test_default_params(product_lib):
    p = L.default_params()
    assert (p.n, p.N, p.k, p.pbs_base_log, p.pbs_level, p.ks_base_log, p.ks_level) == \
        (880, 2048, 1, 23, 1, 3, 5)
    assert p.max_variance_budget == 4000.0


def test_evaluation_key_sizes_and_validation(product_lib):
    """lv_keys_size (host only): BSK n*2*2*N words, KSK N*5*(n+1) words;
    Context.evaluation rejects wrongly sized keys before touching a device."""
    import ctypes
    p = L.default_params()
    nb, nk = ctypes.c_uint64(), ctypes.c_uint64()
    assert product_lib.lv_keys_size(ctypes.byref(p), ctypes.byref(nb), ctypes.byref(nk)) == 0
    assert (nb.value, nk.value) == (880 * 2 * 2 * 2048, 2048 * 5 * 881)
    import numpy as np
    with pytest.raises(L.InvalidParams):
        L.Context.evaluation(np.zeros(7, np.uint64), np.zeros(nk.value, np.uint64), 0)


def test_context_rejects_bad_params(product_lib):
    """Parameter validation happens before any device work (InvalidParams)."""
    for field, value in (("N", 1024), ("k", 2), ("pbs_base_log", 22), ("ks_level", 4), ("n", 0),
                         ("n", 5000), ("lwe_noise_log2", 63), ("glwe_noise_log2", 0),
                         ("exact_mask_product", 3), ("max_variance_budget", 0.5)):
        p = L.default_params()
        setattr(p, field, value)
        with pytest.raises(L.InvalidParams):
            L.Context(seed=0, params=p)


def _band(case):
    m, n = len(case["a"]), len(case["b"])
    mode = case["mode"]
    if mode == "exact":
        return L.BandSpec.exact(m, n)
    if mode == "skip":
        return L.BandSpec.skip(m, n)
    return L.BandSpec.approx(case["ell"])


def test_plan_traces_match_reference_observer(golden, product_lib):
    for tr in golden["traces"]:
        cells, tot = L.plan_trace(len(tr["a"]), len(tr["b"]), _band(tr), tr["key_encoding"],
                                  tr["budget"])
        assert cells == tr["cells"], (tr["a"], tr["b"], tr["budget"])


def test_plan_counters_match_reference_runs(golden, product_lib):
    for case in golden["cases"]:
        m, n = len(case["a"]), len(case["b"])
        if "error" in case:
            if case["error"] == "BandTooNarrow":
                with pytest.raises(L.BandTooNarrow):
                    L.plan_trace(m, n, _band(case), case["key_encoding"], case["budget"])
            if case["error"] == "InvalidParams":
                with pytest.raises(L.InvalidParams):
                    L.plan_trace(m, n, _band(case), case["key_encoding"], case["budget"])
            continue
        rep = case["report"]
        _, tot = L.plan_trace(m, n, _band(case), case["key_encoding"], case["budget"])
        assert tot.visited_cells == rep["visited_cells"]
        assert tot.refreshes == rep["refresh_count"]
        assert tot.max_key_variance == rep["max_key_variance"]


def test_plan_cfg5_maxima(golden, product_lib):
    # every distinct grid shape of cfg5; the worst key is 1780
    seen = {}
    for p in golden["configs"]["cfg5"]:
        m, n = len(p["a"]), len(p["b"])
        if (m, n) not in seen:
            _, tot = L.plan_trace(m, n, L.BandSpec.exact(m, n), "negated", 4000.0)
            seen[(m, n)] = tot
        tot = seen[(m, n)]
        assert tot.max_key_variance == p["report"]["max_key_variance"]
        assert tot.visited_cells == p["report"]["visited_cells"]
        assert tot.refreshes == 0
    assert max(t.max_key_variance for t in seen.values()) == 1780


def test_plan_256_grid_closed_form(product_lib):
    # test_kernel.cpp:367-378: (1 + 4 + 9) * 255 + 1 at 256x256, no refresh
    _, tot = L.plan_trace(256, 256, L.BandSpec.exact(256, 256), "negated", 4000.0)
    assert tot.max_key_variance == 14 * 255 + 1 and tot.refreshes == 0


def test_band_helpers():
    assert L.band_cell_count(100, 10) == 1990
    assert L.BandSpec.skip(15, 15).half_width == 8
    with pytest.raises(L.OutOfRangeValue):
        L.band_cell_count(5, 6)
