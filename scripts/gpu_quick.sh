# Quick perf check: several bench variants (no tests, no profiles).
cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$*', 'value=%.0f'%d['value'], 'step_us=%.1f'%(d['ms_per_step']*1e3), d['step_breakdown_us'], 'frac=%.3f'%d['roofline']['frac'], 'ctx=%d'%d['cache']['contexts'])"; }
for args in "${@}"; do run $args; done
