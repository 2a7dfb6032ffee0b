#!/bin/bash
# Round-2 pass B: the whole GPU suite (no -x), then context-depth sweeps of configs 3 and 2.
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputest_b.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest_b.log
tail -8 gpurun_out/gputest_b.log
bash scripts/sweep_k.sh 3 "16:0 24:12 32:16"
bash scripts/sweep_k.sh 2 "20:0 32:16"
