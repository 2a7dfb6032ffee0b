cd $GRAFT_REPO_ROOT
for se in 8 1000; do for c in 2 3 5; do timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --no-north-star --steps 400 --sample-every $se 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('c$c se=$se', 'value=%.0f'%d['value'], 'step_us=%.1f'%(d['ms_per_step']*1e3), 'fill_mean=%.1f'%d['step_breakdown_us']['roofline_kernel_mean'])"; done; done
