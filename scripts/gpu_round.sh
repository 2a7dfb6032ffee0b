# Full GPU check: tests, smoke, default bench, batch-1024 bench, launch list + ncu full of FillKernel at batch 1024.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ "${TESTS:-1}" = "1" ]; then
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.txt
fi
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --batch 1024 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench1024.json 2>&1; echo "bench1024 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench1024.json')); print('b1024 value', int(d['value']), d['step_breakdown_us'], 'frac', round(d['roofline']['frac'],3))"
if [ "${PROFILE:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2050 -c 100 --csv --log-file gpurun_out/launches.csv python bench.py --steps 60 --warmup 40 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > /dev/null 2>&1; echo "ncu list rc=$?"
python scripts/launches.py gpurun_out/launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:FillKernel -s 2050 -c 1 -o gpurun_out/prof_fill1024 -f python bench.py --batch 1024 --steps 20 --warmup 60 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/ncu_full.log 2>&1; echo "ncu fill rc=$?"
fi
