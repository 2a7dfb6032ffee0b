#!/bin/bash
# Round-2 GPU pass: full GPU suite, then the default bench line.
cd "$GRAFT_REPO_ROOT" || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "bench rc=$?" >> gpurun_out/bench_c3.err
tail -5 gpurun_out/gputest.log
