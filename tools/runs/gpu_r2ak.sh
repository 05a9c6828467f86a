#!/bin/bash
# round 2, call AK: leaf verification out of line -- GPU suite, A/B vs 44f04bc,
# dead-leaf counts
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2ak_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2ak_gpu_tests.log; tail -3 gpurun_out/r2ak_gpu_tests.log
timeout 1200 bash tools/ab_bench.sh r2ak_verify_outline scratch/libbdeg_44f04bc.so -
timeout 300 python tools/sweep_inner.py c5 3 | cut -c1-300
