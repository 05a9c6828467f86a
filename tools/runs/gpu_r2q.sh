#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -q -x -k "not twins" > gpurun_out/r2q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_tests.log
tail -2 gpurun_out/r2q_tests.log
bash tools/ab_bench.sh early scratch/libbdeg_cur.so -
