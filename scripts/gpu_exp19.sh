cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp19
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/exp19/pytest.txt 2>&1; tail -2 gpurun_out/exp19/pytest.txt
VARIANTS="orig base" CONFIGS="3 2 4" STEPS=300 bash scripts/gpu_ab.sh > gpurun_out/exp19/ab.txt 2>&1
grep value= gpurun_out/exp19/ab.txt
