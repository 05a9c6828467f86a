#!/bin/bash
# round 2, call E: sharded walk, exact Smith at scale, integer-pipe peaks v2
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/intpipe_bench tools/intpipe_bench.cu && /tmp/intpipe_bench > gpurun_out/r2e_intpipe.json
cat gpurun_out/r2e_intpipe.json
timeout 900 python -m pytest tests/test_gpu_walk_sharded.py tests/test_gpu_parity_r2.py -q -x -k "sharded or smith or int128" --durations=10 > gpurun_out/r2e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_tests.log
tail -30 gpurun_out/r2e_tests.log
python - > gpurun_out/r2e_f4.log 2>&1 <<'PY'
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
cat gpurun_out/r2e_f4.log
