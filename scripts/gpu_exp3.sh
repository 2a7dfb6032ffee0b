cd $GRAFT_REPO_ROOT
export PRE3_GMASK_LIB=$PWD/paper_2506_03887_b200/libpre3gmask_red.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layout.py -x -q -p no:cacheprovider 2>&1 | tail -3
unset PRE3_GMASK_LIB
VARIANTS="base red" CONFIGS="3 2 4" STEPS=300 bash scripts/gpu_ab.sh
