# Round record: GPU tests, smoke, bench lines for configs 2-5, launch lists and
# ncu --set full captures of the roofline kernels.  Outputs in gpurun_out/final/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
F=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $F/nvidia_smi.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $F/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -1 $F/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $F/smoke.txt 2>&1; echo "smoke rc=$?"
for c in 2 3 4 5; do timeout 900 python bench.py --config $c > $F/bench_c$c.json 2> $F/bench_c$c.err; echo "bench c$c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $F/bench_ref_c2.json 2> $F/bench_ref_c2.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 10100 -c 60 --csv --log-file $F/c2_launches.csv python bench.py --steps 40 --warmup 30 --no-e2e --no-cpu-baseline --no-north-star > /dev/null 2>&1; echo "c2 list rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 10100 -c 60 --csv --log-file $F/c3_launches.csv python bench.py --config 3 --steps 40 --warmup 30 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "c3 list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:FillKernel -s 10040 -c 1 -o $F/c2_fill -f python bench.py --steps 10 --warmup 40 --no-e2e --no-cpu-baseline --no-north-star > $F/c2_full.log 2>&1; echo "c2 full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:FillKernel -s 10040 -c 1 -o $F/c3_fill -f python bench.py --config 3 --steps 10 --warmup 40 --no-e2e --no-cpu-baseline > $F/c3_full.log 2>&1; echo "c3 full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:FillKernel -s 10040 -c 1 -o $F/json1024_fill -f python bench.py --batch 1024 --steps 10 --warmup 40 --no-e2e --no-cpu-baseline > $F/j1024_full.log 2>&1; echo "j1024 full rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:FillKernelILi0ELi0E -s 40 -c 1 -o $F/c4_fill -f python bench.py --config 4 --steps 10 --warmup 40 --no-e2e --no-cpu-baseline > $F/c4_full.log 2>&1; echo "c4 full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:FillKernelILi1ELi0E -s 40 -c 1 -o $F/c5_fill -f python bench.py --config 5 --steps 10 --warmup 40 --no-e2e --no-cpu-baseline > $F/c5_full.log 2>&1; echo "c5 full rc=$?"
