#!/bin/bash
# round 2, call AW: planning cost in the e2e (time-to-degree) arm: tier-sampling count 32 / 16 / 8
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for n in 32 16 8 32; do
  BDEG_TIER_SAMPLES=$n timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('samples $n', round(d['ms_per_step'],4), round(d['time_to_degree_ms'],4), d['result']['overflow_reruns'], d['kernel']['tier'])" | tee -a gpurun_out/r2aw_samples.log
done
