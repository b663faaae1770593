"""GPU: the header-only C++ wrapper (include/leuven_b200.hpp) compiles against
the C ABI and passes reference-shaped tests (tests/cpp/test_wrapper.cpp)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    import paper_2508_14568_b200 as L
    if not os.path.exists(L.LIB_PATH):
        L.build()
    exe = str(tmp_path / "test_wrapper")
    cuda_lib = "/usr/local/cuda/lib64"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_wrapper.cpp"), "-o", exe,
                    "-L", os.path.dirname(L.LIB_PATH), "-lleuven_b200", "-L", cuda_lib, "-lcudart",
                    "-Wl,-rpath," + os.path.dirname(L.LIB_PATH), "-Wl,-rpath," + cuda_lib],
                   check=True)
    return exe


def test_wrapper_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


def reference_report_json(rep):
    """cli.cpp:93-107 report_json(report, include_timing=false) of a golden report."""
    keys = ["distance", "mode", "half_width", "visited_cells", "pbs_total", "pbs_equality",
            "pbs_kernel", "refresh_count", "preprocessing_pbs", "max_key_variance"]
    return json.dumps({k: rep[k] for k in keys}, separators=(",", ":"))


@pytest.mark.gpu
def test_wrapper_runs(tmp_path, golden):
    """Also drives the header's pipeline API (AlphabetSpec, encrypt_string,
    distance with an Eq9Provider, distance_batch, cli::compute_report /
    compute_batch / report_json) over the compiled reference's cases."""
    exe = _build(tmp_path)
    cases = tmp_path / "cases.tsv"
    with open(cases, "w") as f:
        for c in golden["cases"]:
            if "error" in c or "\t" in c["a"] + c["b"] or "\n" in c["a"] + c["b"]:
                continue
            rep = dict(c["report"], mode=c["mode"])
            f.write("\t".join([c["a"], c["b"], c["mode"], str(c["ell"] or 0), c["encoding"],
                               repr(float(c["budget"])), c["key_encoding"],
                               "1" if c["preprocess"] else "0", reference_report_json(rep)]) + "\n")
    r = subprocess.run([exe, str(cases)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
