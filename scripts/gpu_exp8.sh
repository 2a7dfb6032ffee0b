cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp8
VARIANTS="orig base compact" CONFIGS="3 2 4" STEPS=300 bash scripts/gpu_ab.sh > gpurun_out/exp8/ab.txt 2>&1
cat gpurun_out/exp8/ab.txt
