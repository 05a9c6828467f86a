#!/bin/bash
# round 2, call Z2: GPU suite after the degree-only bound fix + ncu of the pair-prefilter C5 kernel
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 12 -c 1 -o gpurun_out/r2z_prof_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "not twins" > gpurun_out/r2z2_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2z2_gpu_tests.log; tail -3 gpurun_out/r2z2_gpu_tests.log
