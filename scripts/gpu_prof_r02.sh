#!/bin/bash
# Round-2 profiles: launch lists (ncu timing only) and one --set full capture
# of the fill kernel per config, after a short prewarm (-s skips past it).
# Outputs under gpurun_out/prof/.  Usage: gpu_prof_r02.sh "3 2 5 4"
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/prof
P=gpurun_out/prof
PW=2000
for c in ${1:-3 2 5}; do
  COMMON="--config $c --prewarm-steps $PW --prewarm-batch 1024 --no-e2e --no-cpu-baseline --cold-steps 0 --no-graph --latency-samples 10 --fill-samples 10"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $((PW + 60)) -c 40 --csv \
    --log-file $P/c${c}_launches.csv python bench.py $COMMON --steps 40 --warmup 30 > /dev/null 2>&1
  echo "c$c list rc=$?"; python scripts/launches.py $P/c${c}_launches.csv > $P/c${c}_launches_summary.txt 2>&1; cat $P/c${c}_launches_summary.txt
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:FillKernel -s $((PW + 40)) -c 1 \
    -o $P/c${c}_fill -f python bench.py $COMMON --steps 10 --warmup 40 > $P/c${c}_full.log 2>&1
  echo "c$c full rc=$?"; python scripts/ncu_summary.py $P/c${c}_fill.ncu-rep > $P/c${c}_fill_summary.txt 2>&1; head -14 $P/c${c}_fill_summary.txt
done
