# ncu --set full of the roofline fill kernel of configs 4 and 5 (traffic for
# the bench's roofline.traffic); prewarm kernels (FillKernel<0, 1>) are not
# matched by the demangled-name filter.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
F=gpurun_out/final
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:FillKernelILi0ELi0E -s 40 -c 1 -o $F/c4_fill -f python bench.py --config 4 --steps 10 --warmup 40 --no-e2e --no-cpu-baseline > $F/c4_full.log 2>&1; echo "c4 full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:FillKernelILi1ELi0E -s 40 -c 1 -o $F/c5_fill -f python bench.py --config 5 --steps 10 --warmup 40 --no-e2e --no-cpu-baseline > $F/c5_full.log 2>&1; echo "c5 full rc=$?"
