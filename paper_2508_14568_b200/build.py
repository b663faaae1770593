"""Builds the in-tree CUDA library paper_2508_14568_b200/_build/libleuven_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a only (B200); no JIT cache, no
torch extension machinery: the .so travels with the repo snapshot to the GPU
box. Incremental: each translation unit is rebuilt only when it or a header
changed.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_build")
LIB = os.path.join(OUT, "libleuven_b200.so")
ROOT = os.path.dirname(HERE)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")] + os.environ.get("LVB_NVCC_EXTRA", "").split()
SOURCES = ["kernels.cu", "ks_tc.cu", "context.cu", "wavefront.cu", "ledger.cpp"]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) + \
        [os.path.join(ROOT, "include", "leuven_b200.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, defines=(), out_dir: str = OUT) -> str:
    """defines: extra -D flags for experiment variants (built into out_dir)."""
    os.makedirs(out_dir, exist_ok=True)
    lib = os.path.join(out_dir, "libleuven_b200.so")
    objs = []
    hdrs = _headers()
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(out_dir, src + ".o")
        objs.append(obj)
        if _stale(obj, [path] + hdrs):
            lang = ["-x", "cu"] if src.endswith(".cpp") else []
            cmd = [NVCC] + ARCH + FLAGS + ["-D" + d for d in defines] + lang + ["-c", path, "-o", obj]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
    if _stale(lib, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-lcudart"]
        subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    # python build.py [DEFINE=VAL ...] [--out DIR]
    args = sys.argv[1:]
    out = OUT
    if "--out" in args:
        i = args.index("--out")
        out = args[i + 1]
        args = args[:i] + args[i + 2:]
    print(build(verbose=True, defines=args, out_dir=out))
