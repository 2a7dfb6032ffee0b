cd $GRAFT_REPO_ROOT
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 40 --error-exitcode 9 python scripts/sanitize_run.py sample graph tiny_table refill > gpurun_out/sanitize_racecheck2.txt 2>&1; echo "racecheck rc=$?"; tail -5 gpurun_out/sanitize_racecheck2.txt
timeout 300 python scripts/sample_rate.py 1024 2>&1
