cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python scripts/sanitize_run.py layout_eos_inside two_streams refill; echo plain=$?
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_run.py layout_eos_inside two_streams > gpurun_out/san2_$tool.txt 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/san2_$tool.txt
done
