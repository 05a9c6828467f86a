#!/bin/bash
# round 2, call AJ: cell-walk baseline at HEAD (W36, W45, W37) + ncu of one W45 walk level
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python tools/walk_runs.py w36,w45,w37 > gpurun_out/r2aj_walk.jsonl 2>&1; cut -c1-250 gpurun_out/r2aj_walk.jsonl
timeout 600 bash tools/runs/gpu_prof_walk.sh r2aj > /dev/null 2>&1; ls -la gpurun_out | grep r2aj
