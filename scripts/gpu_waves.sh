cd $GRAFT_REPO_ROOT
for b in 1024 1110 1184 888; do
timeout 600 python bench.py --config 3 --batch $b --no-e2e --no-cpu-baseline --cold-steps 0 --latency-samples 10 --fill-samples 60 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B=$b', 'value=%.3fM'%(d['value']/1e6), 'step_us=%.1f'%(d['ms_per_step']*1e3), 'fill=%.1f'%d['step_breakdown_us']['roofline_kernel']['mean'], 'frac=%.3f'%d['roofline']['frac'])"
done
