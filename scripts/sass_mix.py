"""Instruction mix (executed warp-instructions per SASS opcode) of one kernel in an ncu report.
usage: python scripts/sass_mix.py report.ncu-rep kernel_regex"""
import csv
import subprocess
import sys
from collections import Counter

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--kernel-name", "regex:" + sys.argv[2]],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
h = rows[hdr]
si, ie, ws = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
c, st = Counter(), Counter()
for r in rows[hdr + 1:]:
    if len(r) <= ie or not r[ie].replace(".", "").isdigit():
        continue
    toks = r[si].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    c[op] += int(float(r[ie]))
    st[op] += int(float(r[ws] or 0))
tot = sum(c.values()) or 1
for op, n in c.most_common(30):
    print(f"{op:12s} {n:14d} {100 * n / tot:5.1f}%  stall_samples={st[op]}")
print("total", tot)
