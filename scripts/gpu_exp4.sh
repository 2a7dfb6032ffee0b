cd $GRAFT_REPO_ROOT
VARIANTS="base red2 nomix" CONFIGS="3 2" STEPS=300 bash scripts/gpu_ab.sh 2>&1 | sort | uniq
timeout 300 python bench.py --config 2 --no-e2e --no-cpu-baseline --cold-steps 0 --latency-samples 10 --fill-samples 32 --no-snapshot | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2 no-snapshot step', d['ms_per_step']*1e3, 'fill', d['step_breakdown_us']['roofline_kernel'])"
timeout 300 python scripts/trace_step.py --split --grammar schema --k 16 --slots 16384 --batch 1024 --prewarm 10000 --per-sm --queue --steps 2
