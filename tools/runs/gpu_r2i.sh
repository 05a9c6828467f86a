#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python tools/sweep_inner.py c5 2,3,4,5 > gpurun_out/r2i_sweep.jsonl 2>&1
timeout 1200 python tools/sweep_inner.py w25,w26 4,5,6 >> gpurun_out/r2i_sweep.jsonl 2>&1
cat gpurun_out/r2i_sweep.jsonl | cut -c1-200
