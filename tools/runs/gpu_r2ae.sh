#!/bin/bash
# round 2, call AE: leaf pivot columns prefetched one leaf ahead -- GPU suite (incl. the nearly-affine
# lifting test), A/B vs 44f04bc
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2ae_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2ae_gpu_tests.log; tail -3 gpurun_out/r2ae_gpu_tests.log
timeout 1200 bash tools/ab_bench.sh r2ae_prefetch scratch/libbdeg_44f04bc.so -
