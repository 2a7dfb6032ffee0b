cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layout.py -q -x -k "sample or Sample" -p no:cacheprovider 2>&1 | tail -1
timeout 600 python scripts/gpu_sample_check.py 64 20 2>&1 | tail -1
timeout 300 python scripts/sample_rate.py 256 1024 2>&1
