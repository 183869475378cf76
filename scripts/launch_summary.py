#!/usr/bin/env python
import csv
import sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = {}
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg.setdefault(r[ki][:60], []).append(float(r[vi].replace(",", "")))
for k, v in agg.items():
    print(f"{k:60s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.1f} us")
