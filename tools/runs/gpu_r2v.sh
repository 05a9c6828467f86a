#!/bin/bash
# round 2, call V: evidence at HEAD (tests, smoke, benches, Table 3 enumeration)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "not twins" > gpurun_out/r2v_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_gpu_tests.log; tail -3 gpurun_out/r2v_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2v_smoke.log 2>&1; cat gpurun_out/r2v_smoke.log
timeout 600 python bench.py > gpurun_out/r2v_bench_c5.json 2> gpurun_out/r2v_bench_c5.err; tail -c 300 gpurun_out/r2v_bench_c5.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2v_bench_reference.json 2>&1
timeout 600 python bench.py --workload w26 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2v_bench_w26.json 2>&1; tail -c 200 gpurun_out/r2v_bench_w26.json
bash tools/runs/gpu_r2p.sh
cp gpurun_out/r2p_table3_enum.jsonl gpurun_out/r2v_table3_enum.jsonl
