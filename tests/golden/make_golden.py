"""Generates tests/golden/*.json from the REFERENCE's own simulated backend.

Run in the build container (needs /root/reference to build oracle/_ref):
    make -C oracle ref && python tests/golden/make_golden.py
The JSON it writes is committed; the GPU box never reads /root/reference.
Every value comes from the compiled reference (proj/src/*.cpp) through
oracle/ref_driver.cpp — nothing here is computed by our own code.
"""
from __future__ import annotations

import ctypes
import json
import random
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2508_14568_b200 import workloads as W  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "libleuven_ref.so")


class Report(ctypes.Structure):
    _fields_ = [
        ("distance", ctypes.c_int32),
        ("half_width", ctypes.c_uint64),
        ("visited_cells", ctypes.c_uint64),
        ("pbs_total", ctypes.c_uint64),
        ("pbs_equality", ctypes.c_uint64),
        ("pbs_kernel", ctypes.c_uint64),
        ("refresh_count", ctypes.c_uint64),
        ("preprocessing_pbs", ctypes.c_uint64),
        ("max_key_variance", ctypes.c_int64),
        ("linear_ops", ctypes.c_uint64),
        ("wall_time_ms", ctypes.c_double),
    ]


ERRORS = {1: "OutOfRangeValue", 2: "NoiseBudgetExceeded", 3: "ValueOutsideLutHalf",
          4: "PackingViolation", 5: "CharNotInAlphabet", 6: "CharNotInSubset",
          7: "PositionOutOfRange", 8: "BandTooNarrow", 9: "FormatError", 10: "InvalidParams"}


def load():
    L = ctypes.CDLL(REF)
    L.ref_compute.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64,
                              ctypes.c_char_p, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                              ctypes.POINTER(Report)]
    L.ref_last_error.restype = ctypes.c_char_p
    L.ref_trace.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64,
                            ctypes.c_char_p, ctypes.c_double, ctypes.c_int, ctypes.c_uint64,
                            ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int64),
                            ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64)]
    L.ref_lut.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
    L.ref_sim_pbs.restype = ctypes.c_double
    L.ref_sim_pbs.argtypes = [ctypes.POINTER(ctypes.c_int32), ctypes.c_uint64, ctypes.c_int,
                              ctypes.POINTER(ctypes.c_int32)]
    L.ref_banded_distance.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64,
                                      ctypes.POINTER(ctypes.c_int32)]
    L.ref_eq_cost.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
    return L


def compute(L, a, b, mode="exact", ell=0, encoding="ascii7", budget=4000.0, key="negated",
            preprocess=False):
    r = Report()
    rc = L.ref_compute(a.encode("latin1"), b.encode("latin1"), mode.encode(), ell,
                       encoding.encode(), budget, 1 if key == "negated" else 0,
                       1 if preprocess else 0, ctypes.byref(r))
    case = {"a": a, "b": b, "mode": mode, "ell": ell, "encoding": encoding, "budget": budget,
            "key_encoding": key, "preprocess": preprocess}
    if rc != 0:
        case["error"] = ERRORS.get(rc, "Error")
        return case
    case["report"] = {f: getattr(r, f) for f, _ in Report._fields_ if f != "wall_time_ms"}
    return case


def trace(L, a, b, mode="exact", ell=0, encoding="ascii7", budget=4000.0, key="negated"):
    cap = (len(a) + 1) * (len(b) + 1)
    ij = (ctypes.c_uint32 * (2 * cap))()
    kv = (ctypes.c_int64 * cap)()
    rf = (ctypes.c_uint32 * cap)()
    cnt = ctypes.c_uint64()
    rc = L.ref_trace(a.encode("latin1"), b.encode("latin1"), mode.encode(), ell,
                     encoding.encode(), budget, 1 if key == "negated" else 0, cap, ij, kv, rf,
                     ctypes.byref(cnt))
    assert rc == 0, L.ref_last_error()
    n = cnt.value
    return {"a": a, "b": b, "mode": mode, "ell": ell, "encoding": encoding, "budget": budget,
            "key_encoding": key,
            "cells": [[ij[2 * t], ij[2 * t + 1], kv[t], rf[t]] for t in range(n)]}


def main():
    L = load()
    out = {"source": "reference SimBackend (proj/src), driven by oracle/ref_driver.cpp"}

    luts = {}
    buf = (ctypes.c_int32 * 16)()
    for name, arg in (("minlut-original", 0), ("minlut-negated", 0), ("identity", 0)):
        assert L.ref_lut(name.encode(), arg, buf) == 0
        luts[name] = list(buf)
    for scale in (1, 9):
        assert L.ref_lut(b"eqlut", scale, buf) == 0
        luts[f"eqlut{scale}"] = list(buf)
    out["luts"] = luts

    # Worked examples and edge cases from the reference's own tests
    # (test_kernel.cpp:230-249, 276-284, 341-352; test_smoke.py:15-55;
    # acceptance main.cpp:138-143).
    cases = [
        ("monday", "friday", {}), ("KID", "SIT", {}), ("abcx", "xabc", {}),
        ("zzzz", "zzzz", {"mode": "skip"}), ("", "", {}), ("abc", "", {}), ("", "abcd", {}),
        ("ab", "", {"mode": "skip"}), ("AAAA", "AAAA", {"mode": "approx", "ell": 0}),
        ("AXBY", "AZBW", {"mode": "approx", "ell": 0}), ("GATT", "ACA", {"encoding": "dna4"}),
        ("kitten", "sitting", {"mode": "skip"}),
        ("abbey", "abbes", {"encoding": "lower26", "preprocess": True}),
        ("k" * 20, "k" * 20, {"budget": 25.0}), ("q" * 30, "q" * 30, {"budget": 25.0}),
        ("XYZ", "ACG", {"encoding": "dna4"}), ("abcdefgh", "ab", {"mode": "approx", "ell": 2}),
        ("ab", "cd", {"budget": 10.0}), ("monday", "friday", {"key": "original"}),
        ("abcdefghijkl", "abxdefhijkzl", {"budget": 11.0}),
        ("querty", "qwerty", {"encoding": "lower26", "preprocess": True}),
        ("ACGTACGTAC", "ACGGTACTAC", {"encoding": "dna4", "preprocess": True}),
        ("monday", "friday", {"mode": "approx", "ell": 2}),
        ("Leuvenshtein", "Levenshtein", {"mode": "skip"}),
    ]
    r = W.MT19937(2024)
    for t in range(24):
        m, n = 1 + r() % 12, 1 + r() % 12
        a = "".join(W.printable(r) for _ in range(m))
        b = ("".join(W.printable(r) for _ in range(n)) if t % 2 else W.mutate(a, r() % 4, r))
        opts = [{}, {"mode": "skip"}, {"mode": "approx", "ell": 3}, {"key": "original"}][t % 4]
        if opts.get("mode") == "skip" and len(b) != len(a):
            opts = {}
        cases.append((a, b, opts))
    for t in range(8):
        m, n = 1 + r() % 10, 1 + r() % 10
        a = "".join(W.dna(r) for _ in range(m))
        b = "".join(W.dna(r) for _ in range(n))
        cases.append((a, b, {"encoding": "dna4", "preprocess": bool(t % 2)}))
    out["cases"] = [compute(L, a, b, **o) for a, b, o in cases]

    # The five BASELINE.json configs (SURVEY §8(d) generator).
    cfgs = {}
    a, b = W.cfg1()
    cfgs["cfg1"] = compute(L, a, b)
    vals = W.cfg2()
    arr = (ctypes.c_int32 * len(vals))(*vals)
    res = (ctypes.c_int32 * len(vals))()
    L.ref_sim_pbs(arr, len(vals), 1, res)
    h = 0
    for v in vals:
        h = (h * 31 + v) & 0xFFFFFFFF
    cfgs["cfg2"] = {"count": len(vals), "message_hash": h, "outputs": list(res)}
    a, b = W.cfg3()
    cfgs["cfg3"] = compute(L, a, b)
    a, b = W.cfg4()
    cfgs["cfg4"] = compute(L, a, b, encoding="dna4", preprocess=True)
    cfgs["cfg5"] = [compute(L, a, b) for a, b in W.cfg5()]
    out["configs"] = cfgs

    # Per-cell traces pinning key variances and refresh placement.
    out["traces"] = [
        trace(L, "m" * 12, "m" * 12),
        trace(L, "m" * 12, "m" * 12, key="original"),
        trace(L, "q" * 30, "q" * 30, budget=25.0),
        trace(L, "abcdefghijkl", "abxdefhijkzl", budget=11.0),
        trace(L, *W.cfg3()),
        trace(L, "kitten", "sitting", mode="approx", ell=2),
        trace(L, "monday", "friday", mode="skip"),
    ]
    # plaintext helpers of the pybind surface (module.cpp:47-108)
    v = ctypes.c_int32()
    out["eq_cost"] = {t: [(L.ref_eq_cost(t.encode(), b, ctypes.byref(v)), v.value)[1]
                          for b in range(1, 65)]
                      for t in ("standard_2bit", "ours_4bit", "combined")}
    rng = random.Random(55)
    banded = []
    for _ in range(40):
        a = "".join(rng.choice("abcdxyz") for _ in range(rng.randint(0, 12)))
        b = "".join(rng.choice("abcdxyz") for _ in range(rng.randint(0, 12)))
        hw = rng.randint(0, 12)
        rc = L.ref_banded_distance(a.encode(), b.encode(), hw, ctypes.byref(v))
        banded.append({"a": a, "b": b, "half_width": hw,
                       "distance": v.value if rc == 0 else None,
                       "error": None if rc == 0 else rc})
    out["banded"] = banded
    # long single pairs: 300 x 300 printable with 40 substitutions (refreshes
    # start at the default budget), and a 256 x 256 skip-band DNA pair
    rng = random.Random(7)
    a = "".join(chr(32 + rng.randrange(95)) for _ in range(300))
    bl = list(a)
    for _ in range(40):
        i = rng.randrange(len(bl))
        bl[i] = chr(32 + rng.randrange(95))
    long_cases = [compute(L, a, "".join(bl))]
    a = "".join(rng.choice("ACGT") for _ in range(256))
    bl = list(a)
    for _ in range(30):
        i = rng.randrange(len(bl))
        bl[i] = rng.choice("ACGT")
    long_cases.append(compute(L, a, "".join(bl), mode="skip", encoding="dna4"))
    out["long"] = long_cases
    path = os.path.join(HERE, "reference_runs.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
