"""Top CUDA source lines by warp-stall samples from `ncu --page source --csv --print-source cuda`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr_i = [i for i, r in enumerate(rows) if r and r[0] in ("#", "Line")][0]
h = rows[hdr_i]
si = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
items = []
for r in rows[hdr_i + 1:]:
    if len(r) <= si:
        continue
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    if v > 0:
        items.append((v, r[0], r[src].strip()[:110]))
tot = sum(v for v, _, _ in items)
for v, line, s in sorted(items, reverse=True)[:n]:
    print(f"{v/tot*100:5.1f}% L{line}: {s}")
