cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp2
timeout 300 python -m pytest tests/test_gpu_call_sequences.py -x -q -p no:cacheprovider 2>&1 | tail -15
timeout 300 python scripts/fill_timing.py --batch 1024 --grammar schema --k 16 --slots 16384 > gpurun_out/exp2/c3_timing.txt 2>&1; echo rc=$?; cat gpurun_out/exp2/c3_timing.txt
