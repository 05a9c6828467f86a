#!/bin/bash
# round 2, call Y: ncu (full, with source) of the leaf-v2 kernels, C5 and W26
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 12 -c 1 -o gpurun_out/r2y_prof_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 12 -c 1 -o gpurun_out/r2y_prof_w26 python bench.py --workload w26 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | grep r2y
