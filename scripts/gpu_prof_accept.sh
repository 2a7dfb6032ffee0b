# ncu --set full of one steady-state AcceptKernel (config 2 split step), warm caches.
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:AcceptKernel -s 50 -c 1 -o gpurun_out/prof_accept -f python bench.py --steps 20 --warmup 40 --no-e2e --no-cpu-baseline --no-north-star > gpurun_out/ncu_acc.log 2>&1; echo "ncu acc rc=$?"
