"""Aggregates an ncu SASS-page capture by CUDA source line (via nvdisasm -g
of the same binary): samples and top stall reasons per line / per function.
usage: python tools/ncu_lines.py rep.ncu-rep lib.so kernel_substring [N]  (design tool)"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, lib, name = sys.argv[1], sys.argv[2], sys.argv[3]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
recs = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    recs.append((int(r[ix["Address"]], 16), int(r[ix["Warp Stall Sampling (All Samples)"]] or 0),
                 {h: int(r[ix[h]] or 0) for h in stall_cols}))
base = min(a for a, _, _ in recs)
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")]
    sass = ""
    for c in cub:
        out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, c)], capture_output=True, text=True).stdout
        if name in out:
            sass = out
lines = sass.split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith("//-----") and name in l)
off2line = {}
cur = None
for l in lines[start + 1:]:
    if l.startswith("//-----"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
agg = defaultdict(lambda: [0, defaultdict(int)])
tot = 0
for a, s, st in recs:
    key = off2line.get(a - base, "?")
    agg[key][0] += s
    tot += s
    for k, v in st.items():
        agg[key][1][k] += v
src = {}
for key in agg:
    if key and key != "?":
        f, ln = key.split(":")
        for root in ("paper_2508_14568_b200/csrc",):
            p = os.path.join(root, f)
            if os.path.exists(p):
                src[key] = open(p).read().split("\n")[int(ln) - 1].strip()[:60]
for key, (s, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{s / tot:6.3f} {key:16s} {src.get(key, ''):60s} " + " ".join(f"{k[6:]}={v / tot:.3f}" for k, v in top))
