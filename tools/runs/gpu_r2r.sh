#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r2r_bench_c5.json 2> gpurun_out/r2r_bench_c5.err; tail -c 300 gpurun_out/r2r_bench_c5.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2r_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 12 -c 1 -o gpurun_out/r2r_prof_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 12 -c 1 -o gpurun_out/r2r_prof_w26 python bench.py --workload w26 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | grep r2r
