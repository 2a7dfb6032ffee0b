#!/bin/bash
# Round-2 record on the current code: GPU tests, smoke, bench lines (default
# = config 3; configs 2/4/5), the reference arm, launch list + one ncu --set
# full capture of config 2's and config 3's fill.  Outputs in gpurun_out/r02/.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/nvidia_smi.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"; cat $O/bench_default.json
for c in ${CONFIGS:-2 4 5}; do timeout 900 python bench.py --config $c > $O/bench_c$c.json 2> $O/bench_c$c.err; echo "bench c$c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"; cat $O/bench_ref.json
