#!/usr/bin/env python
"""Per-kernel means of an ncu --csv launch list (one row per kernel x metric)."""
import csv
import sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
mi = h.index("Metric Name") if "Metric Name" in h else None
ui = h.index("Metric Unit") if "Metric Unit" in h else None
agg = {}
for r in rows[hdr + 1:]:
    if len(r) > vi:
        key = (r[ki][:70], r[mi] if mi is not None else "gpu__time_duration.sum", r[ui] if ui is not None else "")
        agg.setdefault(key, []).append(float(r[vi].replace(",", "")))
for (k, m, u), v in agg.items():
    print(f"{k:70s} {m:28s} n={len(v):3d} mean={sum(v) / len(v):14.1f} {u}")
