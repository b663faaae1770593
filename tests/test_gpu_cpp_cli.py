"""GPU: examples/leuven_compute.cpp — the reference CLI's `compute`
(cli.cpp:53-119) written in C++ over include/leuven_b200.hpp — reproduces
the compiled reference's reports and exit codes on the golden cases."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIELDS = ["distance", "half_width", "visited_cells", "pbs_total", "pbs_equality", "pbs_kernel",
          "refresh_count", "preprocessing_pbs", "max_key_variance"]
EXIT = {"BandTooNarrow": 3, "CharNotInAlphabet": 2, "CharNotInSubset": 2, "InvalidParams": 2,
        "OutOfRangeValue": 2}


def build_cli(out_dir):
    import paper_2508_14568_b200 as L
    if not os.path.exists(L.LIB_PATH):
        L.build()
    exe = os.path.join(str(out_dir), "leuven_compute")
    cuda_lib = "/usr/local/cuda/lib64"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "leuven_compute.cpp"), "-o", exe,
                    "-L", os.path.dirname(L.LIB_PATH), "-lleuven_b200", "-L", cuda_lib, "-lcudart",
                    "-Wl,-rpath," + os.path.dirname(L.LIB_PATH), "-Wl,-rpath," + cuda_lib],
                   check=True)
    return exe


def test_cli_compiles(tmp_path):
    assert os.path.exists(build_cli(tmp_path))


@pytest.mark.gpu
def test_cli_matches_reference_cases(tmp_path, golden):
    exe = build_cli(tmp_path)
    cases = [c for i, c in enumerate(golden["cases"])
             if i < 14 or c["preprocess"] or c.get("error")]
    assert len(cases) >= 20
    for c in cases:
        args = [exe, "--a", c["a"], "--b", c["b"], "--mode", c["mode"], "--encoding", c["encoding"],
                "--budget", repr(c["budget"]), "--key-encoding", c["key_encoding"], "--json"]
        if c["mode"] == "approx":
            args += ["--ell", str(c["ell"])]
        if c["preprocess"]:
            args.append("--preprocess")
        r = subprocess.run(args, capture_output=True, text=True, timeout=300)
        if c.get("error"):
            assert r.returncode == EXIT[c["error"]], (c, r.stderr)
            continue
        assert r.returncode == 0, (c, r.stderr)
        rep = json.loads(r.stdout)
        assert {k: rep[k] for k in FIELDS} == {k: c["report"][k] for k in FIELDS}, c
        assert rep["mode"] == c["mode"]
