cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_layout.py tests/test_gpu_parity.py -k "layout or columns or graph or acceptance or binding or beyond or golden" > gpurun_out/gputest_b.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_b.log
tail -3 gpurun_out/gputest_b.log
TAG=_w300 bash scripts/sweep_k.sh 3 "16:0 32:16" --warmup 300 --steps 120
TAG=_cap64 bash scripts/sweep_k.sh 3 "16:0 32:16" --warmup 300 --steps 120 --stack-cap 64
TAG=_w300 bash scripts/sweep_k.sh 2 "20:0 32:16" --warmup 300 --steps 120
