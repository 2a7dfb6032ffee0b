cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp10
timeout 300 python scripts/fill_timing.py --graph-first 300 > gpurun_out/exp10/c2.txt 2>&1; cat gpurun_out/exp10/c2.txt
timeout 300 python bench.py --config 2 --no-e2e --no-cpu-baseline --cold-steps 0 --fill-samples 40 --no-graph > gpurun_out/exp10/c2_nograph.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/exp10/c2_nograph.json').read().strip().splitlines()[-1]); print('bench c2 no-graph step', d['ms_per_step']*1e3, 'fill', d['step_breakdown_us']['roofline_kernel'])"
