# Quick sweep: context depth and warm-up length (steady state).
cd $GRAFT_REPO_ROOT
for K in 8 12 16; do
  for W in 30 1500; do
    timeout 300 python bench.py --context-depth $K --warmup $W --steps 300 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('K=$K W=$W', 'value=%.0f'%d['value'], 'fill_us=%.1f'%d['mask_latency_us'], 'frac=%.3f'%d['roofline']['frac'], d['cache'])"
  done
done
