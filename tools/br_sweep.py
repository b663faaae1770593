"""Blind-rotation time vs wave size for the single-CTA and CTA-pair kernels
(LVB_BR_PAIR_MAX forces the choice). Prints one JSON line per (variant, count)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_14568_b200 as L  # noqa: E402

counts = [int(x) for x in (sys.argv[1:] or "1 8 24 64 74 100 148 296 444 4096".split())]
for name, pm in (("single", "0"), ("pair", str(1 << 30))):
    os.environ["LVB_BR_PAIR_MAX"] = pm
    ctx = L.Context(seed=0)
    lid = ctx.lut(L.identity_lut())
    for n in counts:
        cts = ctx.encrypt([i % 16 for i in range(n)])
        br, ks, st = ctx.bench_pbs(cts, [lid] * n, 4)
        b = float(np.min(br[1:]))
        print(json.dumps({"variant": name, "count": n, "br_ms": round(b, 3),
                          "pbs_per_s": round(n / b * 1e3, 1)}), flush=True)
        ctx.release(cts)
    ctx.close()
