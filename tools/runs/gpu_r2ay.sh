#!/bin/bash
# round 2, call AY: the GPU suite and smoke at the final HEAD
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2ay_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2ay_gpu_tests.log; tail -3 gpurun_out/r2ay_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ay_smoke.log 2>&1; tail -2 gpurun_out/r2ay_smoke.log
