import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2508_14568_b200 as L
from paper_2508_14568_b200 import workloads as W
c = L.Context(seed=0)
vals = W.cfg2()
h = c.encrypt(vals)
ids = np.full(len(vals), c.lut(L.identity_lut()), np.uint32)
for n in (444, 888, 3552, 3996, 4096, 4440):
    hh = h if n <= 4096 else np.concatenate([h, h[:n - 4096]])
    ii = np.full(n, ids[0], np.uint32)
    br, ks, st = c.bench_pbs(hh[:n], ii, 3)
    print(n, "br_ms", float(np.min(br)), "per item us", float(np.min(br)) * 1e3 / n, flush=True)
