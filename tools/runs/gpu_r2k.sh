#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not twins" > gpurun_out/r2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_tests.log
tail -3 gpurun_out/r2k_tests.log
bash tools/ab_bench.sh pair scratch/libbdeg_cur.so -
