"""Per-phase clock of the throughput blind rotation (diagnostic build with
-DLVB_PROBE, loaded via LVB_LIB): mean SM cycles per CMUX between probe
marks, per warp of CTA 0, on the 4096-item cfg2 batch. (design tool)"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_14568_b200 as L  # noqa: E402
from paper_2508_14568_b200 import workloads as W  # noqa: E402

NAMES = ["decompose", "fwd pass A", "xchg A->B", "pass B", "trip 1", "pass C", "trip 2",
         "pass D", "MAC", "pass D'", "trip C'", "pass C'", "trip B'", "pass B'",
         "bar+xchg B'->A'", "pass A'", "untwist+torus+update"]
count = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
c = L.Context(seed=0)
lib = ctypes.CDLL(os.environ["LVB_LIB"])
buf = (ctypes.c_ulonglong * 128)()
vals = W.cfg2()[:count]
h = c.encrypt(vals)
ids = np.full(len(vals), c.lut(L.identity_lut()), np.uint32)
c.bench_pbs(h, ids, 2)
lib.lv_debug_probe(buf)
br, _, _ = c.bench_pbs(h, ids, 1)
lib.lv_debug_probe(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(4, 32).astype(np.float64)
ncmux = 880 - 1  # CMUXes with a nonzero rotation are ~all; marks count per CMUX
print("BR ms", br, "items", count)
# the CTA-pair kernel (small waves) adds mark 18 (spectrum sent, partner's received) after 8
order = list(range(18)) if count > 148 else [0, 1, 2, 3, 4, 5, 6, 7, 8, 18, 9] + list(range(10, 18))
names = dict(enumerate(["decompose"] + NAMES[1:8] + ["MAC"] + NAMES[9:]))
if count <= 148:
    names[8] = "send + partner wait"
    names[18] = "MAC"
tot = np.zeros(4)
for k0, k1 in zip(order[:-1], order[1:]):
    d = (a[:, k1] - a[:, k0]) / ncmux
    tot += d
    print(f"{k0:2d}->{k1:2d} {names[k0]:24s} " + " ".join(f"{x:7.0f}" for x in d))
print("sum", " ".join(f"{x:7.0f}" for x in tot))
