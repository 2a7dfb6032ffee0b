cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp18
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layout.py tests/test_gpu_bench_parity.py -q -x -k "greedy or tie or special or Greedy or c5 or config5" -p no:cacheprovider 2>&1 | tail -2
VARIANTS="packed base" CONFIGS="5" STEPS=300 bash scripts/gpu_ab.sh > gpurun_out/exp18/ab.txt 2>&1
grep value= gpurun_out/exp18/ab.txt
