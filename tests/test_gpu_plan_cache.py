"""GPU: the traversal-plan cache is LRU-bounded by total cells (ADVICE r1:
a server scanning many string lengths must not grow it without limit).
Run in a subprocess with LVB_PLAN_CACHE_CELLS=40 so every new grid shape
evicts the previous ones (and the largest is never cached); every distance
must still equal Wagner-Fischer, twice over (cold and after eviction)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import paper_2508_14568_b200 as L
from paper_2508_14568_b200 import leuven as LV
ctx = L.Context(seed=5)
pairs = [("kitten", "sitting"), ("ab", "abc"), ("flaw", "lawn"), ("abcdefgh", "abdcefhg"),
         ("", "xyz"), ("gumbo", "gambol")]
for rep in range(2):
    for a, b in pairs:
        r = L.compute(a, b, ctx=ctx)
        assert r["distance"] == LV.wf_distance(a, b) % 32, (a, b, r["distance"])
print("ok")
"""


@pytest.mark.gpu
def test_plan_cache_eviction_keeps_results():
    env = dict(os.environ, LVB_PLAN_CACHE_CELLS="40")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], capture_output=True,
                       text=True, timeout=600, env=env)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
