"""Summarise an ncu --set full report: headline metrics + SASS regions by stalls/instructions."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_write.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for name, val in zip(h, v):
    if name in want:
        print(f"{name:60s} {val}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hh, R = rows[1], rows[2:]
si, ie = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
tot = sum(float(x[si] or 0) for x in R) or 1
ti = sum(float(x[ie] or 0) for x in R) or 1
print(f"SASS lines {len(R)}  stall samples {tot:.0f}  instructions {ti:.0f}")
B = int(sys.argv[2]) if len(sys.argv) > 2 else 100
for b in range(0, len(R), B):
    seg = R[b:b + B]
    s = sum(float(x[si] or 0) for x in seg)
    n = sum(float(x[ie] or 0) for x in seg)
    if s / tot > 0.02 or n / ti > 0.02:
        print(f"  sass {b:5d}-{b + B:5d} stall {s / tot * 100:5.1f}% inst {n / ti * 100:5.1f}%  {seg[0][1].strip()[:60]}")
