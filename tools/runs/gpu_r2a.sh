#!/bin/bash
# round 2, call A: integer-pipe peaks, GPU test suite, smoke, short bench
set -x
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/intpipe_bench tools/intpipe_bench.cu && /tmp/intpipe_bench > gpurun_out/r2a_intpipe.json
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_gpu_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r2a_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
tail -3 gpurun_out/r2a_gpu_tests.log
cat gpurun_out/r2a_intpipe.json
