#!/bin/bash
# round 2, call AA: evidence at HEAD after the leaf rewrite + non-singular counting
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2aa_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2aa_gpu_tests.log; tail -3 gpurun_out/r2aa_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2aa_smoke.log 2>&1; tail -3 gpurun_out/r2aa_smoke.log
timeout 600 python bench.py > gpurun_out/r2aa_bench_c5.json 2> gpurun_out/r2aa_bench_c5.err; tail -c 300 gpurun_out/r2aa_bench_c5.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2aa_bench_reference.json 2>&1
timeout 600 python bench.py --workload w26 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2aa_bench_w26.json 2>&1; tail -c 200 gpurun_out/r2aa_bench_w26.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2aa_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 12 -c 1 -o gpurun_out/r2aa_prof_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 12 -c 1 -o gpurun_out/r2aa_prof_w26 python bench.py --workload w26 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 bash tools/runs/gpu_r2p.sh > /dev/null 2>&1; cp gpurun_out/r2p_table3_enum.jsonl gpurun_out/r2aa_table3_enum.jsonl; cut -c1-250 gpurun_out/r2aa_table3_enum.jsonl
