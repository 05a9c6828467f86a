#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/intpipe_bench tools/intpipe_bench.cu && /tmp/intpipe_bench > gpurun_out/r2g_intpipe.json
cat gpurun_out/r2g_intpipe.json
bash tools/ab_bench.sh leafskip scratch/libbdeg_base.so scratch/libbdeg_leafskip.so scratch/libbdeg_leafskip_mb4.so
