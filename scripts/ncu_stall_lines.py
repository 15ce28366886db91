"""Per-source-line stall breakdown (one stall reason) of an ncu report.
usage: python scripts/ncu_stall_lines.py report.ncu-rep [reason ...]  (reasons: long_sb short_sb wait mio ...)"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, cur, res = None, None, []
for r in rows:
    if len(r) == 2:
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        h = r
        continue
    if h is None or len(r) < len(h) or r[2] != "-":
        continue
    d = dict(zip(h, r))
    res.append((d, (cur or "").split("/")[-1].split("(")[0][-40:] + ":" + r[0], r[1][:90]))


def f(d, k):
    try:
        return float(d.get(k) or 0)
    except ValueError:
        return 0.0


for reason in sys.argv[2:] or ["long_sb", "short_sb", "wait"]:
    key = "stall_" + reason
    tot = sum(f(d, key) for d, _, _ in res) or 1
    print("==", reason)
    for d, loc, src in sorted(res, key=lambda x: -f(x[0], key))[:8]:
        print(f"  {f(d, key) / tot * 100:5.1f}% {loc} {src}")
