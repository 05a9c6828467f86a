#!/bin/bash
# round 2, call Z: non-singular counting + paired half-warp leaf pre-filter -- GPU parity suite, then
# A/B against 2bdb555 (leaf v2) and the same tree at 5 CTAs/SM
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not twins" > gpurun_out/r2z_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2z_gpu_tests.log; tail -3 gpurun_out/r2z_gpu_tests.log
timeout 1200 bash tools/ab_bench.sh r2z_pair scratch/libbdeg_2bdb555.so - scratch/libbdeg_pair_mb5.so
