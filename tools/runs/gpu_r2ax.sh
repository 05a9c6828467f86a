#!/bin/bash
# round 2, call AX: register-DFS depth sweep with the lifting-sorted system plans
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python tools/sweep_inner.py w25 4,5,6 > gpurun_out/r2ax_sweep.jsonl 2>&1
timeout 900 python tools/sweep_inner.py w26 5,6,7 >> gpurun_out/r2ax_sweep.jsonl 2>&1
SWEEP_FLAGS=0x40 timeout 900 python tools/sweep_inner.py w27 6,7 >> gpurun_out/r2ax_sweep.jsonl 2>&1
cut -c1-160 gpurun_out/r2ax_sweep.jsonl
