#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_cache.py -q -p no:cacheprovider -x > gpurun_out/gputest_cache.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_cache.log; tail -15 gpurun_out/gputest_cache.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputest_f.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest_f.log; tail -4 gpurun_out/gputest_f.log
VARIANTS="base" CONFIGS="3 2" bash scripts/gpu_ab.sh 2>&1 | grep -v "^\s\|Traceback\|json.decoder\|File " | head -2
