cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/exp16
for c in 3 2; do for ol in "" "--one-launch"; do
timeout 300 python bench.py --config $c $ol --no-e2e --no-cpu-baseline --cold-steps 0 --latency-samples 10 --fill-samples 16 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c$c $ol', 'value=%.3fM'%(d['value']/1e6), 'step_us=%.1f'%(d['ms_per_step']*1e3), 'fill=%.1f'%d['step_breakdown_us']['roofline_kernel']['mean'], d['launch'] if 'launch' in d else '')"
done; done
