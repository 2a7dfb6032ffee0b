# Lean perf check: bench (no e2e / cpu baseline) + one ncu --set full capture of the fill kernel.
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', int(d['value']), d['step_breakdown_us'], 'frac', round(d['roofline']['frac'],3))"
if [ "${PROFILE:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:FillKernel -s 450 -c 1 -o gpurun_out/prof_fill -f python bench.py --steps 20 --warmup 60 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/ncu_full.log 2>&1; echo "ncu fill rc=$?"
fi
