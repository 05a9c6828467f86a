#!/bin/bash
# round 2, call AV: long walk regressions with the lifting-sorted system plans (N > 64: W_{4,6}/W_{6,4}, W_{3,8}/W_{8,3})
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
BDEG_LONG=1 timeout 2400 python -m pytest tests/test_gpu_parity_r2.py -q -x -k "twins" > gpurun_out/r2av_twins.log 2>&1; echo "rc=$?" >> gpurun_out/r2av_twins.log; tail -3 gpurun_out/r2av_twins.log
