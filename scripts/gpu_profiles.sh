# Round profiles: launch lists (ncu timing only) and one --set full capture per
# dominant kernel.  Outputs under gpurun_out/prof/ (copied to profiles/ by hand).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
P=gpurun_out/prof
# config 2 default (one-launch step, B=256): launch list
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2050 -c 60 --csv --log-file $P/c2_launches.csv python bench.py --steps 40 --warmup 30 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "c2 list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:FillKernel -s 2040 -c 1 -o $P/c2_fill -f python bench.py --steps 10 --warmup 40 --no-e2e --no-cpu-baseline > $P/c2_full.log 2>&1; echo "c2 full rc=$?"
# config 3 (schema, B=1024, separate): launch list + fill kernel full capture
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2050 -c 60 --csv --log-file $P/c3_launches.csv python bench.py --config 3 --steps 40 --warmup 30 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "c3 list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:FillKernel -s 2040 -c 1 -o $P/c3_fill -f python bench.py --config 3 --steps 10 --warmup 40 --no-e2e --no-cpu-baseline > $P/c3_full.log 2>&1; echo "c3 full rc=$?"
# config 2 shape at B=1024 separate (json): fill kernel full capture
timeout 900 ncu --set full --clock-control none --import-source on -k regex:FillKernel -s 2040 -c 1 -o $P/json1024_fill -f python bench.py --batch 1024 --steps 10 --warmup 40 --no-e2e --no-cpu-baseline > $P/j1024_full.log 2>&1; echo "j1024 full rc=$?"
