#!/bin/bash
# round 2, call AB: register-DFS depth sweep at the round-2 leaf; cell-dead detection on slot 0 only (A/B)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python tools/sweep_inner.py c5,w25 2,3,4,5 > gpurun_out/r2ab_sweep_inner.jsonl 2>&1
timeout 900 python tools/sweep_inner.py w26 4,5,6,7 >> gpurun_out/r2ab_sweep_inner.jsonl 2>&1
cut -c1-160 gpurun_out/r2ab_sweep_inner.jsonl
timeout 900 bash tools/ab_bench.sh r2ab_deadslot0 - scratch/libbdeg_deadslot0.so
