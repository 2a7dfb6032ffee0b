#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for k in 4 12; do timeout 300 python scripts/debug_long.py $k 40 2>&1 | tail -2; done
timeout 600 python -m pytest tests/test_gpu_cache.py -q -p no:cacheprovider > gpurun_out/gputest_cache.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_cache.log; tail -4 gpurun_out/gputest_cache.log
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_cache.py -q -p no:cacheprovider -x > gpurun_out/memcheck_cache.txt 2>&1
grep -E "Invalid|ERROR SUMMARY|passed|failed" gpurun_out/memcheck_cache.txt | head -12
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputest_d.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest_d.log; tail -4 gpurun_out/gputest_d.log
bash scripts/gpu_sanitize.sh
