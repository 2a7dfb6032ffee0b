# ncu of the temperature/top-k/top-p step (SampleKernel) at 1,024 JSON sequences.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/prof
timeout 900 ncu --set full --clock-control none --import-source on -k regex:SampleKernel -s 30 -c 1 -o gpurun_out/prof/sample -f \
  python scripts/sample_rate.py 1024 > gpurun_out/prof/sample_full.log 2>&1; echo "full rc=$?"
python scripts/ncu_summary.py gpurun_out/prof/sample.ncu-rep > gpurun_out/prof/sample_summary.txt 2>&1; head -14 gpurun_out/prof/sample_summary.txt
