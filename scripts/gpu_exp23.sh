cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp23
export PRE3_GMASK_LIB=$PWD/paper_2506_03887_b200/libpre3gmask_pad3.so
timeout 600 ncu --metrics launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__shared_mem_per_block_dynamic,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:FillKernel -s 2060 -c 2 python bench.py --config 3 --prewarm-steps 2000 --no-e2e --no-cpu-baseline --cold-steps 0 --no-graph --latency-samples 10 --fill-samples 10 --steps 10 --warmup 40 2>&1 | grep -E "occupancy|shared_mem|duration|warps_active" | head -12
