"""Traversal time of the latency-bound configs cfg1 / cfg3 / cfg4 (second of
two runs each) through compute()."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_14568_b200 as L  # noqa: E402
from paper_2508_14568_b200 import workloads as W  # noqa: E402

ctx = L.Context(seed=0)
for name, fn, kw in (("cfg1", W.cfg1, {}), ("cfg3", W.cfg3, {}),
                     ("cfg4", W.cfg4, {"encoding": "dna4", "preprocess": True})):
    a, b = fn()
    L.compute(a, b, ctx=ctx, **kw)
    t0 = time.perf_counter()
    r = L.compute(a, b, ctx=ctx, **kw)
    dt = time.perf_counter() - t0
    print(f"{name}: {dt * 1e3:.1f} ms, {r['visited_cells'] / dt:.0f} cells/s, distance {r['distance']}",
          flush=True)
