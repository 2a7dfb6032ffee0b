#!/bin/bash
# Stationarity of the synthetic streams: configs 2-5 at 300 steps, stack capacity 1024 vs 64.
cd "$GRAFT_REPO_ROOT" || exit 1
for c in 3 2 5 4; do
  for cap in 64 1024; do
    timeout 900 python bench.py --config $c --stack-cap $cap --steps 300 --warmup 30 --no-e2e --no-cpu-baseline \
      --cold-steps 0 --latency-samples 10 --fill-samples 10 > gpurun_out/depth_c${c}_cap${cap}.json 2> gpurun_out/depth_c${c}_cap${cap}.err
    python - $c $cap <<'PY'
import json, sys
c, cap = sys.argv[1:3]
try:
    d = json.load(open(f"gpurun_out/depth_c{c}_cap{cap}.json"))
    print(f"c{c} cap{cap}: {d['value']/1e6:.3f}M step {d['ms_per_step']*1e3:.1f}us frac {d['roofline']['frac']:.3f} "
          f"walks/seqstep {d['cache']['last_fill']['cd_walks']/8/d['config']['batch_per_gpu']:.1f} depth {d['max_stack_depth_seen']} "
          f"restarts {d['totals']['restarts']} ctx {d['cache']['contexts']} prewarm {d['preprocessing']['prewarm_s']:.1f}s")
except Exception as e:
    print(f"c{c} cap{cap}: failed {e}")
PY
  done
done
