#!/bin/bash
# round 2, call Z4: leaf v2 + non-singular counting (+ last-row pivot fast path) -- GPU parity suite,
# then A/B: 2bdb555 (leaf v2), this tree without the fast pivot, this tree
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not twins" > gpurun_out/r2z4_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2z4_gpu_tests.log; tail -3 gpurun_out/r2z4_gpu_tests.log
timeout 1200 bash tools/ab_bench.sh r2z4_fastpiv scratch/libbdeg_2bdb555.so scratch/libbdeg_nofastpiv.so -
