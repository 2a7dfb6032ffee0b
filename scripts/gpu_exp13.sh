cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp13
VARIANTS="base cgreedy" CONFIGS="5" STEPS=300 bash scripts/gpu_ab.sh > gpurun_out/exp13/ab.txt 2>&1
grep value= gpurun_out/exp13/ab.txt
