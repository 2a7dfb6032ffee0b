#!/bin/bash
# New cache tests, the whole GPU suite, then the default bench line.
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 600 python -m pytest tests/test_gpu_cache.py -q -p no:cacheprovider > gpurun_out/gputest_cache.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_cache.log; tail -15 gpurun_out/gputest_cache.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputest_c.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest_c.log; tail -4 gpurun_out/gputest_c.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c3.json'))
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cold_cache']['mean'], d['check']['equal'], d['max_stack_depth_seen'], d['preprocessing']['prewarm_s'])"
