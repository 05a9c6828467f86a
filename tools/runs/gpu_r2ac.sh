#!/bin/bash
# round 2, call AC: lazy slot 1 at the leaf parents + slot-0 cell-dead test -- GPU parity suite, A/B vs 44f04bc
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2ac_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2ac_gpu_tests.log; tail -3 gpurun_out/r2ac_gpu_tests.log
timeout 1200 bash tools/ab_bench.sh r2ac_lazy1 scratch/libbdeg_44f04bc.so -
