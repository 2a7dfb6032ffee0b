cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp7
VARIANTS="orig base" CONFIGS="3 2 4 5" STEPS=300 bash scripts/gpu_ab.sh > gpurun_out/exp7/ab.txt 2>&1
cat gpurun_out/exp7/ab.txt
