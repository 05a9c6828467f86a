#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python tools/sweep_inner.py w25,w26 4,5,6 > gpurun_out/r2t_sweep.jsonl 2>&1
timeout 1200 python tools/sweep_inner.py c5 3,4 >> gpurun_out/r2t_sweep.jsonl 2>&1
cut -c1-160 gpurun_out/r2t_sweep.jsonl
