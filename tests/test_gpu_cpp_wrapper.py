"""GPU: the header-only C++ wrapper (include/leuven_b200.hpp) compiles against
the C ABI and passes reference-shaped tests (tests/cpp/test_wrapper.cpp)."""
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


@pytest.mark.gpu
def test_wrapper_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
