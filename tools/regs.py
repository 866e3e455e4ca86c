"""Registers / spills per kernel from a libholo build log (ptxas -v):
python tools/regs.py [build.log] [name-filter]"""
import re
import subprocess
import sys

log = sys.argv[1] if len(sys.argv) > 1 else "paper_2004_04049_b200/build.log"
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
rows = []
for ln in open(log):
    m = re.search(r"Compiling entry function '([^']+)'", ln)
    if m:
        cur = [m.group(1), None, None]
        continue
    m = re.search(r"(\d+) bytes spill stores", ln)
    if m and cur:
        cur[2] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", ln)
    if m and cur:
        cur[1] = int(m.group(1))
        rows.append(cur)
        cur = None
names = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True, text=True).stdout.split("\n")
for (mn, reg, sp), dn in zip(rows, names):
    dn = dn.replace("holo::", "").replace("(anonymous namespace)::", "")
    if flt in dn:
        print(f"{reg:4d} regs {sp or 0:4d} B spill  {dn[:150]}")
