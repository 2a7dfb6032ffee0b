cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp21
VARIANTS="ipc8 ipc7" CONFIGS="2 3 5" STEPS=300 bash scripts/gpu_ab.sh > gpurun_out/exp21/ab.txt 2>&1
grep value= gpurun_out/exp21/ab.txt
