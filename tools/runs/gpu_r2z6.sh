#!/bin/bash
# round 2, call Z6: V-only, one-slot walk of cell-dead subtrees -- GPU parity suite, A/B against 44f04bc
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not twins" > gpurun_out/r2z6_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2z6_gpu_tests.log; tail -3 gpurun_out/r2z6_gpu_tests.log
timeout 1200 bash tools/ab_bench.sh r2z6_deadv scratch/libbdeg_44f04bc.so -
