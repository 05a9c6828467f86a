#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python tools/sweep_inner.py w26 6,7 > gpurun_out/r2u_sweep.jsonl 2>&1
SWEEP_FLAGS=0x40 timeout 1200 python tools/sweep_inner.py w27 6,7 >> gpurun_out/r2u_sweep.jsonl 2>&1
timeout 1200 python tools/sweep_inner.py w27 6,7 >> gpurun_out/r2u_sweep.jsonl 2>&1
cut -c1-170 gpurun_out/r2u_sweep.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "inner_levels or systems_full or table3" > gpurun_out/r2u_tests.log 2>&1; tail -2 gpurun_out/r2u_tests.log
