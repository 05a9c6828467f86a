#!/bin/bash
# round 2, call AP: point-order sweep on master-space workloads (W25, W26): kernel time per order
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python tools/order_sweep.py w25,w26 > gpurun_out/r2ap_order_sweep.jsonl 2>&1; cut -c1-200 gpurun_out/r2ap_order_sweep.jsonl
