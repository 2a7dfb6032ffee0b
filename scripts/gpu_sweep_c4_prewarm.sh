cd $GRAFT_REPO_ROOT
run() { timeout 600 python bench.py --config 4 --no-e2e --no-cpu-baseline --steps 300 "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$*', 'value=%.0f'%d['value'], 'step_us=%.1f'%(d['ms_per_step']*1e3), 'fill_p50=%.1f'%d['step_breakdown_us']['roofline_kernel_p50'], 'frac=%.3f'%d['roofline']['frac'], 'ctx', d['preprocessing']['contexts_after_prewarm'], '->', d['cache']['contexts'], 'prewarm_s=%.1f'%d['preprocessing']['prewarm_s'])"; }
run
run --prewarm-steps 30000
run --prewarm-steps 30000 --context-slots 262144
run --prewarm-steps 50000 --context-slots 262144
