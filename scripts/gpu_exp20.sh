cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp20
VARIANTS="base r56" CONFIGS="3 2 5 4" STEPS=300 bash scripts/gpu_ab.sh > gpurun_out/exp20/ab.txt 2>&1
grep value= gpurun_out/exp20/ab.txt
