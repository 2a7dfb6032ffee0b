#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over every
# device step form (scripts/sanitize_run.py), logs in gpurun_out/sanitize_*.txt.
cd "$GRAFT_REPO_ROOT" || exit 1
CS=/usr/local/cuda/bin/compute-sanitizer
python scripts/sanitize_run.py > gpurun_out/sanitize_plain.txt 2>&1; echo "plain rc=$?" >> gpurun_out/sanitize_plain.txt
for tool in memcheck synccheck racecheck initcheck; do
  parts=""
  [ "$tool" = racecheck ] && parts="two_call split split_two_grid greedy sample graph tiny_table refill parents overflow layout_eos_inside two_streams"
  timeout 1500 $CS --tool $tool --print-limit 40 --error-exitcode 9 python scripts/sanitize_run.py $parts \
    > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.txt
  tail -3 gpurun_out/sanitize_$tool.txt
done
