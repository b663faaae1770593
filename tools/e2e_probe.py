"""e2e (host buffers) vs device timing of cfg2 through lv_pbs_batch_host."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_14568_b200 as L
from paper_2508_14568_b200 import workloads as W
c = L.Context(seed=0)
vals = W.cfg2()
h = c.encrypt(vals)
ids = np.full(len(vals), c.lut(L.identity_lut()), np.uint32)
rows = c.export(h)
pin_in = torch.from_numpy(rows).pin_memory(); pin_out = torch.empty_like(pin_in).pin_memory()
a, b = pin_in.numpy(), pin_out.numpy()
for _ in range(2): c.pbs_host(a, ids, b)
torch.cuda.synchronize()
for _ in range(3):
    t = time.perf_counter(); c.pbs_host(a, ids, b); dt = time.perf_counter() - t
    print(f"e2e {dt*1e3:.1f} ms -> {len(vals)/dt:.0f} PBS/s")
br, ks, st = c.bench_pbs(h, ids, 3)
print("device step ms", list(st))
