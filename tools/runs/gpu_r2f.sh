#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -q -x -k "not twins and not smith" > gpurun_out/r2f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_tests.log
tail -5 gpurun_out/r2f_tests.log
bash tools/ab_bench.sh depmask scratch/libbdeg_base.so -
