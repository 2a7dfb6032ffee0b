#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_cache.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "cache or overlay or pushing or snapshot or idle or greedy" > gpurun_out/gputest_e.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_e.log; tail -5 gpurun_out/gputest_e.log
VARIANTS="base" CONFIGS="3 2 5" bash scripts/gpu_ab.sh 2>&1 | grep -v "^\s\|Traceback\|json.decoder\|File "
