#!/bin/bash
# round 2, call D: full GPU suite, f4 timing, launch list + ncu --set full of C5 and W26 (front end)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 -k "not twins" > gpurun_out/r2d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_tests.log
tail -32 gpurun_out/r2d_tests.log
python - > gpurun_out/r2d_f4.log 2>&1 <<'PY'
import time, json, sys
sys.path.insert(0, ".")
import torch, workloads as W, paper_1501_02237_b200 as B
torch.cuda.set_device(0)
for mm in (10, 20, 30, 40):
    A, b = W.master_space_system(mm, mm)
    B.smith_gpu(A); B.dimension_modp(A)
    t0 = time.perf_counter(); r = B.smith_gpu(A); t1 = time.perf_counter()
    d = B.dimension_modp(A); t2 = time.perf_counter()
    print(json.dumps({"m": mm, "k": mm, "n": len(A), "m_eq": len(A[0]), "exact_rank": r[0], "dim": len(A) - r[0],
                      "components": r[1], "unit_pivots": r[2], "smith_gpu_s": t1 - t0, "dim_modp": d,
                      "dimension_modp_2primes_s": t2 - t1}), flush=True)
PY
cat gpurun_out/r2d_f4.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 9 -c 1 -o gpurun_out/r2d_prof_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 9 -c 1 -o gpurun_out/r2d_prof_w26 python bench.py --workload w26 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 python bench.py --workload w26 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_bench_w26.json 2>&1; tail -c 600 gpurun_out/r2d_bench_w26.json
ls -la gpurun_out
