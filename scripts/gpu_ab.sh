#!/bin/bash
# A/B of library variants on one box: VARIANTS="base v1 ..." CONFIGS="2 3 ..." [STEPS=] [EXTRA=]
# (variants built by scripts/build_variant.sh NAME "-D..."; base = the in-tree library).
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in ${VARIANTS}; do
  if [ "$v" = "base" ]; then unset PRE3_GMASK_LIB; else export PRE3_GMASK_LIB=$PWD/paper_2506_03887_b200/libpre3gmask_$v.so; fi
  for c in ${CONFIGS:-2 3 5}; do
    timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --cold-steps 0 --latency-samples 10 \
      --fill-samples 16 --steps ${STEPS:-200} ${EXTRA:-} 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$v c$c', 'value=%.3fM'%(d['value']/1e6), 'step_us=%.1f'%(d['ms_per_step']*1e3), 'fill_mean=%.1f'%d['step_breakdown_us']['roofline_kernel']['mean'], 'frac=%.3f'%d['roofline']['frac'], 'ok=%s'%d['check'].get('equal'))" || echo "$v c$c failed"
  done
done
done
