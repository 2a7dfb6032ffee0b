cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp5
VARIANTS="base nomix red2 lsu" CONFIGS="3 2" STEPS=300 bash scripts/gpu_ab.sh > gpurun_out/exp5/ab.txt 2>&1
cat gpurun_out/exp5/ab.txt
