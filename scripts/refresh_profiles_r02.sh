#!/bin/bash
# Copies a gpu_final_r02.sh run into profiles/ as the round-2 record.
set -e
cd "$(dirname "$0")/.."
F=gpurun_out/final2
P=profiles
Q=gpurun_out/prof
for c in 2 3 4 5; do cp $F/bench_c$c.json $P/r02_bench_c$c.json; done
cp $F/bench_ref_c3.json $P/r02_bench_reference_c3.json
cp $F/pytest_gpu.txt $P/r02_pytest_gpu.txt
cp $F/smoke.txt $P/r02_smoke.txt
summ() {  # rep -> summary with stall reasons and top lines
  python scripts/ncu_summary.py $1 2>/dev/null; echo; echo "stall reasons:"
  ncu -i $1 --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]; items=[]
for name,val in zip(h,v):
    if name.startswith('smsp__pcsamp_warps_issue_stalled_') and not name.endswith('_not_issued'):
        try: items.append((float(val.replace(',','')), name))
        except: pass
tot=sum(x for x,_ in items) or 1
for x,n in sorted(items,reverse=True)[:8]: print('  %5.1f%% %s'%(100*x/tot,n.replace('smsp__pcsamp_warps_issue_stalled_','')))
"; echo; echo "top CUDA lines by stall samples:"; python scripts/ncu_cuda_lines.py $1 15
}
for c in 2 3 4 5; do
  cp $Q/c${c}_launches.csv $P/r02_c${c}_launches.csv
  python scripts/launches.py $Q/c${c}_launches.csv > $P/r02_c${c}_launches_summary.txt
  summ $Q/c${c}_fill.ncu-rep > $P/r02_c${c}_fill_summary.txt
done
[ -f $Q/c4_accept.ncu-rep ] && summ $Q/c4_accept.ncu-rep > $P/r02_c4_accept_summary.txt && rm -f $P/r02_c2_accept_summary.txt
summ $Q/sample.ncu-rep > $P/r02_sample_summary.txt
cp $Q/c3_fill.ncu-rep $P/r02_c3_fill.ncu-rep
python - <<'PY'
import json, subprocess, io, csv
def dram(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out))); h, u, v = r[0], r[1], r[2]
    d = dict(zip(h, zip(u, v)))
    def b(k):
        unit, val = d[k]; val = float(val.replace(",", ""))
        return val * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[unit]
    return int(b("dram__bytes_read.sum") + b("dram__bytes_write.sum"))
Q = "gpurun_out/prof"
t = json.load(open("profiles/traffic.json"))
src = "ncu --set full, one steady-state launch (profiles/r02_c%d_fill_summary.txt)"
t["json:128255:256:stream:separate"].update(dram_bytes_per_launch=dram(Q + "/c2_fill.ncu-rep"), source=src % 2)
t["schema:128255:1024:stream:separate"].update(dram_bytes_per_launch=dram(Q + "/c3_fill.ncu-rep"), source=src % 3)
t["sql:128255:4096:stream:separate"].update(dram_bytes_per_launch=dram(Q + "/c4_fill.ncu-rep"), source=src % 4)
g = t.pop("json:128255:512:greedy:fused", {})
g.update(dram_bytes_per_launch=dram(Q + "/c5_fill.ncu-rep"), source=src % 5)
t["json:128255:512:greedy:separate"] = g
json.dump(t, open("profiles/traffic.json", "w"), indent=1)
print(t)
PY
