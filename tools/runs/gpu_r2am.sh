#!/bin/bash
# round 2, call AM: narrow walk elimination two rows per pass -- walk parity tests, walk A/B vs 44f04bc
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "walk" > gpurun_out/r2am_walk_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2am_walk_tests.log; tail -3 gpurun_out/r2am_walk_tests.log
timeout 1500 bash tools/ab_walk.sh r2am_walkrows2 scratch/libbdeg_44f04bc.so -
