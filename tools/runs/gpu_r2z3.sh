#!/bin/bash
# round 2, call Z3: pair pre-filter with single-copy leaf code (points 0..15 in both halves) --
# GPU parity suite, then A/B against 2bdb555 (leaf v2)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not twins" > gpurun_out/r2z3_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2z3_gpu_tests.log; tail -3 gpurun_out/r2z3_gpu_tests.log
timeout 1200 bash tools/ab_bench.sh r2z3_pair1 scratch/libbdeg_2bdb555.so -
