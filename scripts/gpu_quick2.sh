cd $GRAFT_REPO_ROOT
run() { timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-north-star "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$*', 'value=%.0f'%d['value'], 'kern=%.1f'%d['mask_latency_us'], 'frac=%.3f'%d['roofline']['frac'], 'ctx=%d'%d['cache']['contexts'], 'prewarm_s=%.1f'%d['preprocessing']['prewarm_s'], 'pre_ctx=%d'%d['preprocessing']['contexts_after_prewarm'])"; }
for args in "${@}"; do run $args; done
