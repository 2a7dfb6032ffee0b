# Config 2 (K = 20): parent depth and table size.
cd $GRAFT_REPO_ROOT
run() { timeout 600 python bench.py --config 2 --no-e2e --no-cpu-baseline --no-north-star --steps 300 "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$*', 'value=%.0f'%d['value'], 'step_us=%.1f'%(d['ms_per_step']*1e3), 'fill=%.1f'%d['step_breakdown_us']['roofline_kernel_mean'], 'frac=%.3f'%d['roofline']['frac'], 'ctx', d['preprocessing']['contexts_after_prewarm'], '->', d['cache']['contexts'])"; }
run
run --parent-depth 8
run --parent-depth 12
run --context-slots 131072
run --context-depth 20 --prewarm-steps 20000
