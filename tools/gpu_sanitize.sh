#!/bin/bash
# compute-sanitizer over every kernel family (small inputs)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2ao_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r2ao_sanitize_$tool.log
done
