cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp9
VARIANTS="orig base compact rall" CONFIGS="3 2" STEPS=300 bash scripts/gpu_ab.sh > gpurun_out/exp9/ab.txt 2>&1
grep value= gpurun_out/exp9/ab.txt
