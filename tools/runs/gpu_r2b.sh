#!/bin/bash
# round 2, call B: the new parity tests (+ the twins) on the current kernel
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity_r2.py -q -x -k "not twins" --durations=15 > gpurun_out/r2b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_tests.log
tail -25 gpurun_out/r2b_tests.log
BDEG_LONG=1 timeout 1500 python -m pytest tests/test_gpu_parity_r2.py -q -x -k "twins and pair0" --durations=5 > gpurun_out/r2b_twins.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_twins.log
tail -8 gpurun_out/r2b_twins.log
