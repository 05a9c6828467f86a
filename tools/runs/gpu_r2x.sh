#!/bin/bash
# round 2, call X: leaf v2 (cross-product X, relative fp32 keys + CREDUX.MIN.F32, zero prefix columns,
# whole-item instantiations) -- GPU parity suite, then A/B against the HEAD-of-session library
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not twins" > gpurun_out/r2x_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_gpu_tests.log; tail -3 gpurun_out/r2x_gpu_tests.log
timeout 900 bash tools/ab_bench.sh r2x_leafv2 scratch/libbdeg_2bb573e.so -
