#!/bin/bash
# A/B of library variants incl. cold-cache latency: VARIANTS="base v1 ..." CONFIGS="4 2 ..."
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in ${VARIANTS}; do
  if [ "$v" = "base" ]; then unset PRE3_GMASK_LIB; else export PRE3_GMASK_LIB=$PWD/paper_2506_03887_b200/libpre3gmask_$v.so; fi
  for c in ${CONFIGS:-2 3 4}; do
    timeout 900 python bench.py --config $c --no-e2e --no-cpu-baseline --cold-steps 100 --latency-samples 10 \
      --fill-samples 60 --steps ${STEPS:-300} 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$v c$c', 'value=%.3fM'%(d['value']/1e6), 'step_us=%.1f'%(d['ms_per_step']*1e3), 'fill_mean=%.1f'%d['step_breakdown_us']['roofline_kernel']['mean'], 'cold_mean=%.0f'%d['cold_cache']['mean'], 'cold_p50=%.0f'%d['cold_cache']['p50'])" || echo "$v c$c failed"
  done
done
done
