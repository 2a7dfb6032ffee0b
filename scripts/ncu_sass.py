"""Top SASS instructions by warp-stall samples from `ncu --page source --csv` (SASS view)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
items = []
for idx, r in enumerate(rows[hi + 1:]):
    try:
        v = float(r[si] or 0)
    except (ValueError, IndexError):
        continue
    items.append((v, idx, r[0], r[src].strip()[:90]))
tot = sum(v for v, *_ in items) or 1
for v, idx, addr, s in sorted(items, reverse=True)[:n]:
    print(f"{v/tot*100:5.1f}% #{idx:4d} {addr}: {s}")
