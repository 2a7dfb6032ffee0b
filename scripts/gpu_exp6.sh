cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp6
VARIANTS="orig base ipw2 ipw3 ipw4" CONFIGS="3 2 4" STEPS=300 bash scripts/gpu_ab.sh > gpurun_out/exp6/ab.txt 2>&1
cat gpurun_out/exp6/ab.txt
