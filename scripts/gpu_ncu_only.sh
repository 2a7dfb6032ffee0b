cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
F=gpurun_out/final
# ncu --set full captures of the roofline kernels.  Outputs in gpurun_out/final/.
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 10100 -c 60 --csv --log-file $F/c2_launches.csv python bench.py --steps 40 --warmup 30 --no-e2e --no-cpu-baseline --no-north-star > /dev/null 2>&1; echo "c2 list rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 10100 -c 60 --csv --log-file $F/c3_launches.csv python bench.py --config 3 --steps 40 --warmup 30 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "c3 list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:FillKernel -s 10040 -c 1 -o $F/c2_fill -f python bench.py --steps 10 --warmup 40 --no-e2e --no-cpu-baseline --no-north-star > $F/c2_full.log 2>&1; echo "c2 full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:FillKernel -s 10040 -c 1 -o $F/c3_fill -f python bench.py --config 3 --steps 10 --warmup 40 --no-e2e --no-cpu-baseline > $F/c3_full.log 2>&1; echo "c3 full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:FillKernel -s 10040 -c 1 -o $F/json1024_fill -f python bench.py --batch 1024 --steps 10 --warmup 40 --no-e2e --no-cpu-baseline > $F/j1024_full.log 2>&1; echo "j1024 full rc=$?"
