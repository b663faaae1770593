import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2508_14568_b200 as L
ctx = L.Context(seed=0)
lid = ctx.lut(L.identity_lut())
for n in [int(x) for x in (sys.argv[1:] or ["1", "24", "148"])]:
    cts = ctx.encrypt([i % 16 for i in range(n)])
    br, ks, st = ctx.bench_pbs(cts, [lid] * n, 4)
    print(os.environ.get("TAG", ""), n, "br_ms", float(np.min(br[1:])), flush=True)
