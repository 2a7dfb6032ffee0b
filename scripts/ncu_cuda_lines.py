"""Per-CUDA-line stall/instruction shares from `ncu -i REP --page source --csv --print-source cuda,sass`."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hdr]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
items = []
for r in rows[hdr + 1:]:
    if len(r) > ie and r[0] not in ("", "-"):
        try:
            items.append((float(r[si] or 0), float(r[ie] or 0), int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
ts = sum(x[0] for x in items) or 1
ti = sum(x[1] for x in items) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
key = 1 if len(sys.argv) > 3 and sys.argv[3] == "inst" else 0
for s, i, line, src in sorted(items, key=lambda x: -x[key])[:n]:
    print(f"stall {s / ts * 100:5.1f}% inst {i / ti * 100:5.1f}%  L{line}: {src}")
