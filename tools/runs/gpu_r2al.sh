#!/bin/bash
# round 2, call AL: final evidence at HEAD (suite incl. the 4-rank shared queue, smoke, benches)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -s -k "steal" > gpurun_out/r2al_steal.log 2>&1; grep -E "world|passed|failed" gpurun_out/r2al_steal.log | tail -8
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2al_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2al_gpu_tests.log; tail -3 gpurun_out/r2al_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2al_smoke.log 2>&1; tail -2 gpurun_out/r2al_smoke.log
timeout 600 python bench.py > gpurun_out/r2al_bench_c5.json 2> gpurun_out/r2al_bench_c5.err; tail -c 300 gpurun_out/r2al_bench_c5.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2al_bench_reference.json 2>&1; tail -c 200 gpurun_out/r2al_bench_reference.json
timeout 600 python bench.py --workload w26 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2al_bench_w26.json 2>&1; tail -c 200 gpurun_out/r2al_bench_w26.json
