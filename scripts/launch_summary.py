"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel count / total / mean (us)."""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = OrderedDict()
for r in rows[start + 1:]:
    name = r[ki].split("(")[0][:70]
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] == "ns" else (v * 1e3 if r[ui] == "ms" else v)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1; a[1] += v
tot = sum(a[1] for a in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:12.1f} us {100*t/tot:5.1f}%  n={n:3d}  mean={t/n:10.1f} us  {k}")
