# Context depth K sweep (configs 2, 3, 5).
cd $GRAFT_REPO_ROOT
run() { timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-north-star --steps 300 "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$*', 'value=%.0f'%d['value'], 'step_us=%.1f'%(d['ms_per_step']*1e3), 'fill=%.1f'%d['step_breakdown_us']['roofline_kernel_mean'], 'frac=%.3f'%d['roofline']['frac'], 'ctx', d['preprocessing']['contexts_after_prewarm'], '->', d['cache']['contexts'])"; }
for k in 8 12 16 20 24; do run --config 2 --context-depth $k; done
for k in 8 12 16 20; do run --config 3 --context-depth $k; done
for k in 8 12 16; do run --config 5 --context-depth $k; done
