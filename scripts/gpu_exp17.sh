cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp17
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layout.py -q -x -k "sample or Sample" -p no:cacheprovider 2>&1 | tail -2
timeout 600 python scripts/gpu_sample_check.py 64 20 > gpurun_out/exp17/check.txt 2>&1; tail -3 gpurun_out/exp17/check.txt
timeout 300 python scripts/sample_rate.py 256 1024 > gpurun_out/exp17/new.txt 2>&1; cat gpurun_out/exp17/new.txt
