#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not twins" > gpurun_out/r2s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_tests.log
tail -2 gpurun_out/r2s_tests.log
bash tools/ab_bench.sh minblocks scratch/libbdeg_mb3.so scratch/libbdeg_mb5.so -
