cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp11
PRE3_DIAG_FILL_FIRST=1 timeout 300 python bench.py --config 2 --no-e2e --no-cpu-baseline --cold-steps 0 --fill-samples 40 > gpurun_out/exp11/c2.json 2> gpurun_out/exp11/c2.err; grep diag gpurun_out/exp11/c2.err; python -c "
import json; d=json.loads(open('gpurun_out/exp11/c2.json').read().strip().splitlines()[-1]); print('bench c2 step', d['ms_per_step']*1e3, 'fill', d['step_breakdown_us']['roofline_kernel'])"
PRE3_DIAG_FILL_FIRST=1 timeout 300 python bench.py --config 3 --no-e2e --no-cpu-baseline --cold-steps 0 --fill-samples 40 > gpurun_out/exp11/c3.json 2> gpurun_out/exp11/c3.err; grep diag gpurun_out/exp11/c3.err; python -c "
import json; d=json.loads(open('gpurun_out/exp11/c3.json').read().strip().splitlines()[-1]); print('bench c3 step', d['ms_per_step']*1e3, 'fill', d['step_breakdown_us']['roofline_kernel'])"
