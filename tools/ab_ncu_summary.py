"""Summarise gpurun_out/ab_*.csv (tools/ab_ncu.sh): per variant and kernel, mean time and DRAM bytes."""
import csv
import glob
import os
from collections import defaultdict

for f in sorted(glob.glob("gpurun_out/ab_*.csv")):
    rows = list(csv.reader(open(f)))
    try:
        hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    except StopIteration:
        print(os.path.basename(f), "no data")
        continue
    h = rows[hdr]
    ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    d = defaultdict(lambda: defaultdict(list))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1, "msecond": 1,
             "usecond": 1e-3, "nsecond": 1e-6}
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            d[r[ki][:40]][r[mi]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1))
    for k, m in d.items():
        t = sum(m["gpu__time_duration.sum"]) / max(1, len(m["gpu__time_duration.sum"]))
        rd = sum(m["dram__bytes_read.sum"]) / max(1, len(m["dram__bytes_read.sum"]))
        wr = sum(m["dram__bytes_write.sum"]) / max(1, len(m["dram__bytes_write.sum"]))
        print(f"{os.path.basename(f):24s} {k:40s} {t:8.3f} ms  read {rd / 1e9:7.3f} GB  write {wr / 1e9:7.3f} GB")
