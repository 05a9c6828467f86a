#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_tests.log
tail -2 gpurun_out/r2l_tests.log
BDEG_LIB=scratch/libbdeg_redux.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2l_tests_redux.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_tests_redux.log
tail -2 gpurun_out/r2l_tests_redux.log
bash tools/ab_bench.sh split scratch/libbdeg_cur.so scratch/libbdeg_redux.so -
