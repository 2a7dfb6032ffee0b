cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp22
VARIANTS="base pad3" CONFIGS="3 2 5 4" STEPS=300 bash scripts/gpu_ab.sh > gpurun_out/exp22/ab.txt 2>&1
grep value= gpurun_out/exp22/ab.txt
