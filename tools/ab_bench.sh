#!/bin/bash
# A/B of library builds on the same box: bash tools/ab_bench.sh <tag> <lib>...  (a lib "-" = the in-tree build)
# Each build is a git revision compiled into scratch/ (DESIGN.md names the revisions compared).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=$1; shift
for round in 1 2; do
  for lib in "$@"; do
    if [ "$lib" == "-" ]; then unset BDEG_LIB; else export BDEG_LIB=$lib; fi
    for wl in c5 w26; do
      steps=20; [ $wl == w26 ] && steps=3
      out=$(timeout 600 python bench.py --workload $wl --steps $steps --warmup 3 --no-cpu-baseline 2>&1 | tail -1)
      ms=$(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['result']['degree'])" 2>/dev/null)
      echo "$TAG round $round lib $lib $wl: $ms" | tee -a gpurun_out/ab_$TAG.log
    done
  done
done
unset BDEG_LIB
