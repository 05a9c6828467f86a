#!/bin/bash
# round 2, call C: work queue + overflow chain (tier 4): full GPU suite, steal test, bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=20 -k "not twins" > gpurun_out/r2c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_tests.log
tail -30 gpurun_out/r2c_tests.log
timeout 300 python -m pytest tests/test_gpu_steal.py -q -s > gpurun_out/r2c_steal.log 2>&1; tail -8 gpurun_out/r2c_steal.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; tail -c 1500 gpurun_out/r2c_bench.json; tail -3 gpurun_out/r2c_bench.err
