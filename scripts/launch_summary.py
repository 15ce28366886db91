"""Aggregate an ncu --csv launch list: per kernel name, count and mean of each metric."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
agg = defaultdict(lambda: defaultdict(list))
order = []
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")[:60]
    if name not in order:
        order.append(name)
    agg[name][r[mi]].append(float(r[vi].replace(",", "")))
for n in order:
    m = agg[n]
    t = m.get("gpu__time_duration.sum", [0])
    line = f"{n:60s} n={len(t):3d} time={sum(t) / len(t) / 1e3:9.3f} us"
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in m:
            line += f" {k.split('.')[0].split('__')[1]}={sum(m[k]) / len(m[k]) / 1e9:7.3f} GB"
    print(line)
