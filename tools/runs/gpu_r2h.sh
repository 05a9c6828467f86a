#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not twins" > gpurun_out/r2h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_tests.log
tail -3 gpurun_out/r2h_tests.log
bash tools/ab_bench.sh mb4 scratch/libbdeg_base.so -
for wl in w25 w27; do timeout 900 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --degree-only 2>&1 | tail -1 | cut -c1-250; done
