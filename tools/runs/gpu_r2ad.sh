#!/bin/bash
# round 2, call AD: 5 CTAs/SM (96 registers) at HEAD's kernel, A/B
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 bash tools/ab_bench.sh r2ad_mb5 - scratch/libbdeg_head_mb5.so
