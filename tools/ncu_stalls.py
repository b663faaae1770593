"""Top stall sites of an ncu --set full capture (SASS page): instruction,
samples, and the dominant stall reasons; optional opcode aggregation.
usage: python tools/ncu_stalls.py rep.ncu-rep [N] [--ops]   (design tool)"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
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
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    st = {h: int(r[ix[h]] or 0) for h in stall_cols}
    recs.append((s, r[ix["Address"]], r[ix["Source"]].strip(), st, int(r[ix["Instructions Executed"]] or 0)))
tot = sum(x[0] for x in recs)
agg = defaultdict(int)
for x in recs:
    for k, v in x[3].items():
        agg[k] += v
print("total samples", tot)
print("by reason:", ", ".join(f"{k[6:]} {v / tot:.3f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))
if "--ops" in sys.argv:
    ops = defaultdict(lambda: [0, 0])
    for s, a, src, st, n in recs:
        op = src.split()[0] if not src.startswith("@") else src.split()[1]
        op = op.split(".")[0]
        ops[op][0] += s
        ops[op][1] += n
    for op, (s, n) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:30]:
        print(f"{op:12s} samples {s / tot:6.3f}  warp-instr {n}")
    sys.exit()
for s, a, src, st, n in sorted(recs, key=lambda x: -x[0])[:N]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{s / tot:6.3f} {a[-5:]} {src[:60]:60s} " + " ".join(f"{k[6:]}={v}" for k, v in top))
