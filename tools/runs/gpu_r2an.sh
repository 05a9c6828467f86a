#!/bin/bash
# round 2, call AN: narrow walk elimination G rows per pass (G = 2 in-tree, G = 4 scratch) -- walk tests,
# walk A/B (kernel times) vs 44f04bc
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "walk" > gpurun_out/r2an_walk_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2an_walk_tests.log; tail -3 gpurun_out/r2an_walk_tests.log
timeout 1800 bash tools/ab_walk.sh r2an_walkrows scratch/libbdeg_44f04bc.so - scratch/libbdeg_walkrows4.so
