# Config 4: context depth K x parent depth R (30k-step prewarm).
cd $GRAFT_REPO_ROOT
run() { timeout 600 python bench.py --config 4 --no-e2e --no-cpu-baseline --steps 300 "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$*', 'value=%.0f'%d['value'], 'step_us=%.1f'%(d['ms_per_step']*1e3), 'fill=%.1f'%d['step_breakdown_us']['roofline_kernel_mean'], 'frac=%.3f'%d['roofline']['frac'], 'ctx', d['preprocessing']['contexts_after_prewarm'], '->', d['cache']['contexts'])"; }
run --context-depth 20 --parent-depth 6
run --context-depth 22 --parent-depth 6
run --context-depth 24 --parent-depth 6
run --context-depth 24 --parent-depth 8
run --context-depth 18 --parent-depth 6
