# Parent depth R sweep over configs 2-5 (context builds from the context keyed R deep).
cd $GRAFT_REPO_ROOT
run() { timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-north-star --steps 200 "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$*', 'value=%.0f'%d['value'], 'step_us=%.1f'%(d['ms_per_step']*1e3), 'fill_p50=%.1f'%d['step_breakdown_us']['roofline_kernel_p50'], 'frac=%.3f'%d['roofline']['frac'], 'ctx', d['preprocessing']['contexts_after_prewarm'], '->', d['cache']['contexts'], 'prewarm_s=%.1f'%d['preprocessing']['prewarm_s'])"; }
for c in ${CONFIGS:-2 3 4 5}; do for r in ${RS:-4 6 8 10}; do run --config $c --parent-depth $r; done; done
