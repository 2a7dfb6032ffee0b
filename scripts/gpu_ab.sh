# A/B of library variants on one box: VARIANTS="base mb5 ..." CONFIGS="2 3 ...".
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in ${VARIANTS}; do
  if [ "$v" = "base" ]; then unset PRE3_GMASK_LIB; else export PRE3_GMASK_LIB=$PWD/paper_2506_03887_b200/libpre3gmask_$v.so; fi
  for c in ${CONFIGS:-2 3 5}; do
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --no-north-star --steps ${STEPS:-200} ${EXTRA:-} 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$v c$c', 'value=%.0f'%d['value'], 'step_us=%.1f'%(d['ms_per_step']*1e3), 'fill_p50=%.1f'%d['step_breakdown_us']['roofline_kernel_p50'], 'frac=%.3f'%d['roofline']['frac'])"
  done
done
done
