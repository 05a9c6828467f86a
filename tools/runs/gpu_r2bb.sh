#!/bin/bash
# round 2, call BB: final evidence at the residual order: benches, ncu of W26, smoke, long twin walks (N > 64)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bb_smoke.log 2>&1; tail -2 gpurun_out/r2bb_smoke.log
timeout 600 python bench.py > gpurun_out/r2bb_bench_c5.json 2> gpurun_out/r2bb_bench_c5.err; tail -c 300 gpurun_out/r2bb_bench_c5.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2bb_bench_reference.json 2>&1
timeout 600 python bench.py --workload w26 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2bb_bench_w26.json 2>&1; tail -c 200 gpurun_out/r2bb_bench_w26.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 12 -c 1 -o gpurun_out/r2bb_prof_w26 python bench.py --workload w26 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
BDEG_LONG=1 timeout 2400 python -m pytest tests/test_gpu_parity_r2.py -q -x -k "twins" > gpurun_out/r2bb_twins.log 2>&1; echo "rc=$?" >> gpurun_out/r2bb_twins.log; tail -2 gpurun_out/r2bb_twins.log
