#!/bin/bash
# Light-pass phase timelines of the config-2 step (trace_step.py): with logits, without.
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 600 python scripts/trace_step.py --batch 256 --split --k 20 --slots 65536 --prewarm 10000 --steps 2 2>&1 | tail -12
timeout 600 python scripts/trace_step.py --batch 256 --split --k 20 --slots 65536 --prewarm 10000 --steps 1 --no-logits 2>&1 | tail -9
timeout 600 python scripts/trace_step.py --batch 1024 --split --k 16 --grammar schema --slots 16384 --prewarm 10000 --steps 1 2>&1 | tail -9
