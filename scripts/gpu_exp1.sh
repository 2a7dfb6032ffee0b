cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp1
timeout 600 python scripts/fill_timing.py > gpurun_out/exp1/c2_timing.txt 2>&1; echo rc=$?; cat gpurun_out/exp1/c2_timing.txt
timeout 600 python scripts/fill_timing.py --batch 1024 --grammar schema --k 16 --slots 16384 > gpurun_out/exp1/c3_timing.txt 2>&1; echo rc=$?; cat gpurun_out/exp1/c3_timing.txt
P=gpurun_out/exp1
COMMON="--config 2 --prewarm-steps 2000 --prewarm-batch 1024 --no-e2e --no-cpu-baseline --cold-steps 0 --no-graph --latency-samples 10 --fill-samples 10"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2060 -c 40 --csv --log-file $P/c2_launches.csv python bench.py $COMMON --steps 40 --warmup 30 > /dev/null 2>&1
echo "list rc=$?"; python scripts/launches.py $P/c2_launches.csv
