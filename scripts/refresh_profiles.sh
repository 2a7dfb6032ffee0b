# Copies a gpu_final.sh run (gpurun_out/final/) into profiles/ as the round record.
set -e
cd "$(dirname "$0")/.."
F=gpurun_out/final
P=profiles
R=${ROUND:-r01}
for c in 2 3 4 5; do cp $F/bench_c$c.json $P/${R}_bench_c$c.json; done
cp $F/bench_ref_c2.json $P/${R}_bench_reference_c2.json
cp $F/pytest_gpu.txt $P/${R}_pytest_gpu.txt
cp $F/smoke.txt $P/${R}_smoke.txt
for c in c2 c3; do
  cp $F/${c}_launches.csv $P/${R}_${c}_launches.csv
  python scripts/launches.py $F/${c}_launches.csv > $P/${R}_${c}_launches_summary.txt
done
for r in c2_fill c3_fill json1024_fill c4_fill c5_fill; do
  (python scripts/ncu_summary.py $F/$r.ncu-rep 2>/dev/null; echo; echo "stall reasons:";
   ncu -i $F/$r.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]; items=[]
for name,val in zip(h,v):
    if name.startswith('smsp__pcsamp_warps_issue_stalled_') and not name.endswith('_not_issued'):
        try: items.append((float(val.replace(',','')), name))
        except: pass
tot=sum(x for x,_ in items) or 1
for x,n in sorted(items,reverse=True)[:8]: print('  %5.1f%% %s'%(100*x/tot,n.replace('smsp__pcsamp_warps_issue_stalled_','')))
"; echo; echo "top CUDA lines by stall samples:"; python scripts/ncu_cuda_lines.py $F/$r.ncu-rep 15) > $P/${R}_${r}_summary.txt
done
cp $F/c3_fill.ncu-rep $P/${R}_c3_fill.ncu-rep
python - <<'PY'
import json, subprocess, io, csv
def dram(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out))); h, u, v = r[0], r[1], r[2]
    d = dict(zip(h, zip(u, v)))
    def mb(k):
        unit, val = d[k]; val = float(val.replace(",", ""))
        return val * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[unit]
    return int(mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"))
F = "gpurun_out/final"
t = {
 "json:128255:256:stream:separate": {"dram_bytes_per_launch": dram(F + "/c2_fill.ncu-rep"), "source": "ncu --set full, FillKernel<0,0> (profiles/r01_c2_fill_summary.txt)", "note": "at 256 sequences the masked logits (63 MB) mostly stay dirty in the 126 MB L2 when the kernel ends; their write-back is not attributed to the launch, so DRAM writes under-count"},
 "schema:128255:1024:stream:separate": {"dram_bytes_per_launch": dram(F + "/c3_fill.ncu-rep"), "source": "ncu --set full, FillKernel<0,0> (profiles/r01_c3_fill_summary.txt)"},
 "json:128255:1024:stream:separate": {"dram_bytes_per_launch": dram(F + "/json1024_fill.ncu-rep"), "source": "ncu --set full, FillKernel<0,0> (profiles/r01_json1024_fill_summary.txt)"},
 "sql:128255:4096:stream:separate": {"dram_bytes_per_launch": dram(F + "/c4_fill.ncu-rep"), "source": "ncu --set full, FillKernel<0,0> (profiles/r01_c4_fill_summary.txt)"},
 "json:128255:512:greedy:fused": {"dram_bytes_per_launch": dram(F + "/c5_fill.ncu-rep"), "source": "ncu --set full, FillKernel<1,0> (profiles/r01_c5_fill_summary.txt)", "note": "greedy reads only the 16-B logit chunks holding allowed tokens"},
}
json.dump(t, open("profiles/traffic.json", "w"), indent=1)
print(t)
PY
