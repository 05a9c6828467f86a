#!/bin/bash
# round 2, call W: HEAD re-check after the container restart + SASS-level ncu of the C5 / W26 kernels
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2w_bench_c5.json 2> gpurun_out/r2w_bench_c5.err; tail -c 400 gpurun_out/r2w_bench_c5.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 12 -c 1 -o gpurun_out/r2w_prof_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 12 -c 1 -o gpurun_out/r2w_prof_w26 python bench.py --workload w26 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | grep r2w
