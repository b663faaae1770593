"""Lists local-memory spill instructions of one kernel with their source lines.
usage: python tools/spills.py <cubin or .o> <mangled kernel name substring>
(design tool, not part of the product)"""
import re
import subprocess
import sys
import tempfile
import os

obj, name = sys.argv[1], sys.argv[2]
with tempfile.TemporaryDirectory() as d:
    if not obj.endswith(".cubin"):
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                       capture_output=True)
        obj = os.path.join(d, [f for f in os.listdir(d) if f.endswith(".cubin")][0])
    txt = subprocess.run(["nvdisasm", "-g", "-c", obj], capture_output=True, text=True).stdout
lines = txt.split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith("//-----") and name in l)
cur = None
for l in lines[start + 1:]:
    if l.startswith("//-----"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], m.group(2))
    if "STL" in l or "LDL" in l:
        print(cur, l.strip()[:72])
