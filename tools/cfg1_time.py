import time, numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2508_14568_b200 as L
from paper_2508_14568_b200 import workloads as W
ctx = L.Context(seed=0)
a, b = W.cfg1()
spec = L.AlphabetSpec.ascii7()
for it in range(3):
    t0 = time.perf_counter()
    xs = L.encrypt_string(a, spec, ctx); ys = L.encrypt_string(b, spec, ctx)
    t1 = time.perf_counter()
    r = L.distance_encrypted(ctx, xs, ys, L.BandSpec.exact(8, 8))
    t2 = time.perf_counter()
    d = ctx.decrypt([r.score])
    t3 = time.perf_counter()
    print(f"encrypt {1e3*(t1-t0):.2f} ms  traverse {1e3*(t2-t1):.2f} ms  decrypt {1e3*(t3-t2):.2f} ms  waves {r.waves} dist {d[0]}")
