# Sweep: batch x context depth x prewarm length (steady state vs in-run builds).
cd $GRAFT_REPO_ROOT
for B in 256 1024; do
 for K in 8 12 16; do
  for P in 400 2000; do
    timeout 300 python bench.py --batch $B --context-depth $K --prewarm-steps $P --steps 300 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
c=d['cache']
print('B=$B K=$K P=$P', 'value=%.0f'%d['value'], 'fill_us=%.1f'%d['mask_latency_us'], 'step_us=%.1f'%(d['ms_per_step']*1e3), 'frac=%.3f'%d['roofline']['frac'], 'ctx_pre=%d'%d['preprocessing']['contexts_after_prewarm'], 'ctx=%d'%c['contexts'], 'prewarm_s=%.1f'%d['preprocessing']['prewarm_s'], 'walks=%d'%c['last_fill']['cd_walks'])"
  done
 done
done
