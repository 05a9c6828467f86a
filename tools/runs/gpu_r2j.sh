#!/bin/bash
# round 2, call J: evidence at HEAD
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not twins" > gpurun_out/r2j_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_gpu_tests.log; tail -3 gpurun_out/r2j_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; cat gpurun_out/r2j_smoke.log
timeout 600 python bench.py > gpurun_out/r2j_bench_c5.json 2> gpurun_out/r2j_bench_c5.err; tail -c 400 gpurun_out/r2j_bench_c5.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2j_bench_reference.json 2>&1; tail -c 300 gpurun_out/r2j_bench_reference.json
timeout 600 python bench.py --workload w26 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_bench_w26.json 2>&1; tail -c 300 gpurun_out/r2j_bench_w26.json
BDEG_DEBUG=1 timeout 900 python tools/walk_sharded_run.py w45,w37 2 > gpurun_out/r2j_walk_sharded.jsonl 2> gpurun_out/r2j_walk_sharded.err; cat gpurun_out/r2j_walk_sharded.jsonl | cut -c1-400
python - > gpurun_out/r2j_f4.log 2>&1 <<'PY'
import time, json, sys
sys.path.insert(0, ".")
import numpy as np, torch, workloads as W, paper_1501_02237_b200 as B
torch.cuda.set_device(0)
for mm in (10, 20, 30, 40):
    A, b = W.master_space_system(mm, mm)
    An = np.array(A, dtype=np.int64)
    B.smith_gpu(An); B.dimension_modp(An)
    t0 = time.perf_counter(); r = B.smith_gpu(An); t1 = time.perf_counter()
    d = B.dimension_modp(An); t2 = time.perf_counter()
    print(json.dumps({"m": mm, "k": mm, "n": An.shape[0], "m_eq": An.shape[1], "exact_rank": r[0], "dim": An.shape[0] - r[0],
                      "components": r[1], "unit_pivots": r[2], "smith_gpu_s": t1 - t0, "dim_modp": d,
                      "dimension_modp_2primes_s": t2 - t1, "input": "numpy int64 (no list marshalling)"}), flush=True)
PY
cat gpurun_out/r2j_f4.log
BDEG_LONG=1 timeout 1500 python -m pytest tests/test_gpu_parity_r2.py -q -x -k "twins and pair1" --durations=3 > gpurun_out/r2j_twins_w38_w83.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_twins_w38_w83.log; tail -6 gpurun_out/r2j_twins_w38_w83.log
