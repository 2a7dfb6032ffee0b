#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for k in 4 12; do timeout 300 python scripts/debug_long.py $k 40 2>&1 | tail -4; done
timeout 300 python scripts/debug_long.py 4 12 2>&1 | tail -3
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python scripts/debug_long.py 4 40 > gpurun_out/debug_long_memcheck.txt 2>&1
grep -E "Invalid|ERROR SUMMARY|at 0x|by thread" gpurun_out/debug_long_memcheck.txt | head -20
