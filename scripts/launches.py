"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) * scale[r[ui]])
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k[:50]:50s} n={len(v):4d} mean={sum(v)/len(v):8.2f}us min={min(v):8.2f} share={sum(v)/tot*100:5.1f}%")
