cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp15
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layout.py -q -x -k "sample or Sample" -p no:cacheprovider 2>&1 | tail -2
PRE3_GMASK_LIB=$PWD/paper_2506_03887_b200/libpre3gmask_orig.so timeout 300 python scripts/sample_rate.py 1024 > gpurun_out/exp15/orig.txt 2>&1
timeout 300 python scripts/sample_rate.py 256 1024 > gpurun_out/exp15/new.txt 2>&1
echo orig; cat gpurun_out/exp15/orig.txt; echo new; cat gpurun_out/exp15/new.txt
