#!/bin/bash
# Context-depth sweep: bench.py --config C with K:R pairs (reduced run:
# no e2e / CPU baseline / cold steps).  Usage: sweep_k.sh C "16:0 24:8 32:16" [extra bench args]
cd "$GRAFT_REPO_ROOT" || exit 1
C=$1; shift; PAIRS=$1; shift
for kr in $PAIRS; do
  K=${kr%%:*}; R=${kr##*:}; TAG=${TAG:-}
  timeout 900 python bench.py --config "$C" --context-depth "$K" --parent-depth "$R" --steps 60 --warmup 10 \
    --no-e2e --no-cpu-baseline --cold-steps 0 --latency-samples 10 --fill-samples 10 "$@" \
    > "gpurun_out/sweep_c${C}_k${K}_r${R}${TAG}.json" 2> "gpurun_out/sweep_c${C}_k${K}_r${R}${TAG}.err"
  python - "$C" "$K" "$R" "$TAG" <<'PY'
import json, sys
c, k, r, tag = sys.argv[1:5]
try:
    d = json.load(open(f"gpurun_out/sweep_c{c}_k{k}_r{r}{tag}.json"))
    print(f"c{c}{tag} K={k} R={r}: {d['value']/1e6:.3f}M seq-steps/s step {d['ms_per_step']*1e3:.1f}us fill {d['mask_latency_us']:.1f}us "
          f"frac {d['roofline']['frac']:.3f} prewarm {d['preprocessing']['prewarm_s']:.1f}s ctx {d['cache']['contexts']} "
          f"walks/seqstep {d['cache']['last_fill']['cd_walks']/8/d['config']['batch_per_gpu']:.1f} depth {d['max_stack_depth_seen']} "
          f"check {d['check']['token_digest']}")
except Exception as e:
    print(f"c{c} K={k} R={r}: failed {e}")
PY
done
