#!/bin/bash
# round 2, call AG: why the parent certificates do not pay on C5 -- dead-leaf counts and ncu
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python tools/sweep_inner.py c5 3 > gpurun_out/r2ag_sweep.jsonl 2>&1; cat gpurun_out/r2ag_sweep.jsonl | cut -c1-300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 12 -c 1 -o gpurun_out/r2ag_prof_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | grep r2ag
