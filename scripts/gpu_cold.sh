#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for v in "a:" "b:--cold-steps 0" "c:--no-e2e --no-cpu-baseline"; do
  tag=${v%%:*}; args=${v#*:}
  timeout 900 python bench.py $args > gpurun_out/cold_$tag.json 2> gpurun_out/cold_$tag.err
  python - $tag <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/cold_{t}.json"))
    print(t, f"{d['value']/1e6:.3f}M step {d['ms_per_step']*1e3:.1f}us walks/seqstep {d['cache']['last_fill']['cd_walks']/8/1024:.1f} "
          f"depth {d['max_stack_depth_seen']} prewarm {d['preprocessing']['prewarm_s']:.1f}s cold {d.get('cold_cache', {}).get('mean')}")
except Exception as e:
    print(t, "failed", e)
PY
done
