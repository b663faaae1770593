"""Profiling target: 2 x (KS + BR) over the cfg2 batch (used under ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2508_14568_b200 as L
from paper_2508_14568_b200 import workloads as W
count = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
c = L.Context(seed=0)
vals = W.cfg2(count)
h = c.encrypt(vals)
ids = np.full(count, c.lut(L.identity_lut()), np.uint32)
br, ks, st = c.bench_pbs(h, ids, 2)
print("br_ms", list(br), "ks_ms", list(ks))
