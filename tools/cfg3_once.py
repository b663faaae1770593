"""One cfg3 traversal (for a launch list under ncu). (design tool)"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_14568_b200 as L  # noqa: E402
from paper_2508_14568_b200 import workloads as W  # noqa: E402
ctx = L.Context(seed=0)
a, b = W.cfg3()
L.compute(a, b, ctx=ctx)
t0 = time.perf_counter()
r = L.compute(a, b, ctx=ctx)
print("cfg3 ms", (time.perf_counter() - t0) * 1e3, r["distance"], r["waves"])
