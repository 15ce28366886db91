"""Per-source-line executed instructions and stall samples of one kernel in an ncu report.
usage: python scripts/ncu_lines.py report.ncu-rep [top_n]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, res, h = None, [], None
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        h = r
        ie, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
        continue
    if h is None or len(r) <= ie or r[2] != "-":
        continue
    try:
        n = float(r[ie] or 0)
    except ValueError:
        continue
    if n > 0:
        res.append((n, float(r[ws] or 0), (cur or "").split("/")[-1], r[0], r[1][:100]))
res.sort(reverse=True)
tot, stt = sum(o[0] for o in res), sum(o[1] for o in res)
for o in res[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{o[0] / tot * 100:5.1f}% stall={o[1] / stt * 100:5.1f}% {o[2]}:{o[3]} {o[4]}")
