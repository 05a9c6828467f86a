#!/bin/bash
# A/B of library builds on the cell walk: bash tools/ab_walk.sh <tag> <lib>...  (a lib "-" = the in-tree build)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=$1; shift
for round in 1 2; do
  for lib in "$@"; do
    if [ "$lib" == "-" ]; then unset BDEG_LIB; else export BDEG_LIB=$lib; fi
    out=$(timeout 600 python tools/walk_runs.py w36,w36,w45,w37 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print(d['wl'], round(d['walk_s'],3), round(d['kernel_ms']/1e3,3), d['degree'], end='; ')
    except Exception: pass")
    echo "$TAG round $round lib $lib: $out" | tee -a gpurun_out/ab_$TAG.log
  done
done
unset BDEG_LIB
