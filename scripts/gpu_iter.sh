# Iteration check: GPU parity tests, then quick bench lines for configs 2-5
# (no e2e/CPU baseline), then a steady-state trace at batch 256.
cd $GRAFT_REPO_ROOT
if [ "${TESTS:-1}" = "1" ]; then
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.txt
fi
bash scripts/gpu_quick.sh "--config 2 --no-north-star" "--config 2 --batch 1024 --no-north-star" "--config 3" "--config 4" "--config 5"
if [ "${TRACE:-1}" = "1" ]; then
python scripts/trace_step.py --batch 256 --k 16 --slots 65536 --parent 4 --steps 2 --queue --split 2>&1 | grep -v "^ *h:"
fi
