#!/bin/bash
# round 2, call BA: residual-sorted system plans -- GPU suite, A/B vs the lifting-sorted build, Table 3
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2ba_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2ba_gpu_tests.log; tail -3 gpurun_out/r2ba_gpu_tests.log
timeout 1200 bash tools/ab_bench.sh r2ba_residorder scratch/libbdeg_liftorder.so -
timeout 900 bash tools/runs/gpu_r2p.sh > /dev/null 2>&1; cp gpurun_out/r2p_table3_enum.jsonl gpurun_out/r2ba_table3_enum.jsonl; cut -c1-250 gpurun_out/r2ba_table3_enum.jsonl
