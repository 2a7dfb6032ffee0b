#!/bin/bash
# Round-2 record: GPU tests, smoke, bench lines (configs 2-5 + the reference
# arm), then ncu launch lists and --set full captures (gpu_prof_r02.sh) plus
# the accept and sampler kernels.  Outputs in gpurun_out/final2/ and
# gpurun_out/prof/; scripts/refresh_profiles_r02.sh copies them to profiles/.
cd "$GRAFT_REPO_ROOT" || exit 1
F=gpurun_out/final2; mkdir -p $F
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $F/nvidia_smi.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $F/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -1 $F/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $F/smoke.txt 2>&1; echo "smoke rc=$?"
for c in 3 2 4 5; do timeout 900 python bench.py --config $c > $F/bench_c$c.json 2> $F/bench_c$c.err; echo "bench c$c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $F/bench_ref_c3.json 2> $F/bench_ref_c3.err; echo "ref rc=$?"
bash scripts/gpu_prof_r02.sh "3 2 5 4" > $F/prof.log 2>&1; echo "prof rc=$?"
P=gpurun_out/prof
# The separate accept kernel: the split step's two-kernel form at config 4 (the default carries the accepts in the fill's grid).
PRE3_SPLIT_TWO_KERNELS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:AcceptKernel -s 45 -c 1 -o $P/c4_accept -f \
  python bench.py --config 4 --prewarm-steps 2000 --prewarm-batch 1024 --no-e2e --no-cpu-baseline --cold-steps 0 --no-graph \
  --latency-samples 10 --fill-samples 10 --steps 10 --warmup 40 > $P/c4_accept.log 2>&1; echo "accept rc=$?"
bash scripts/gpu_prof_sample.sh > /dev/null 2>&1; echo "sample prof rc=$?"
