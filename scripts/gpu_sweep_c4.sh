cd $GRAFT_REPO_ROOT
for K in 12 20 28 32; do
timeout 600 python bench.py --config 4 --context-depth $K --context-slots 65536 --no-e2e --no-cpu-baseline --steps 100 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
c=d['cache']
print('K=$K', 'value=%.0f'%d['value'], 'step_us=%.1f'%(d['ms_per_step']*1e3), 'frac=%.3f'%d['roofline']['frac'], 'ctx_pre=%d'%d['preprocessing']['contexts_after_prewarm'], 'ctx=%d'%c['contexts'], 'priv=%d'%c['private_builds'], 'prewarm_s=%.1f'%d['preprocessing']['prewarm_s'], 'walks=%d'%c['last_fill']['cd_walks'])"
done
