"""Quick device timing of the cfg2 batched PBS (dev tool, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2508_14568_b200 as L
from paper_2508_14568_b200 import workloads as W
t = time.time()
p = L.default_params()
p.exact_mask_product = int(os.environ.get("QUICK_EXACT", "0"))  # exact-mask keys
c = L.Context(seed=1, params=p)
print("ctx+keygen s", time.time() - t, flush=True)
vals = W.cfg2()
h = c.encrypt(vals)
lid = c.lut(L.identity_lut())
ids = np.full(len(vals), lid, np.uint32)
for count in (int(a) for a in (sys.argv[1:] or ["4096"])):
    br, ks, st = c.bench_pbs(h[:count], ids[:count], 5)
    print(f"count {count}: ks {ks} ms br {br} ms step {st} ms -> {count / (np.median(st) / 1e3):.0f} PBS/s", flush=True)
out = c.pbs(h, lid)
d = c.decrypt(out)
print("correct", int((d == np.array(vals)).sum()), "of", len(vals))
