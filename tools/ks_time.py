"""Key-switch (tcgen05 GEMM) time vs batch size, TMA-fed vs cp.async-fed
(LVB_KS_NO_TMA=1). Prints one JSON line per count."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_14568_b200 as L  # noqa: E402

ctx = L.Context(seed=0)
lid = ctx.lut(L.identity_lut())
for n in [int(x) for x in (sys.argv[1:] or "24 128 512 4096".split())]:
    cts = ctx.encrypt([i % 16 for i in range(n)])
    br, ks, st = ctx.bench_pbs(cts, [lid] * n, 5)
    print(json.dumps({"tma": not os.environ.get("LVB_KS_NO_TMA"), "count": n,
                      "ks_ms": round(float(np.min(ks[1:])), 4)}), flush=True)
    ctx.release(cts)
