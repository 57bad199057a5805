"""Summarise an ncu launch list CSV (gpu__time_duration.sum per launch)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        d[r[ki][:70]].append(float(r[vi].replace(",", "")))
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{k:70s} n={len(v):3d} mean={sum(v) / len(v) / 1e6:8.3f} ms")
