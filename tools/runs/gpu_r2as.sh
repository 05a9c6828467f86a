#!/bin/bash
# round 2, call AS: point orders from the subdivision's vertex set (W25, W26, W27) vs the lifting order
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SWEEP_VERTEX=1 SWEEP_ORDERS=planner,lift_asc,vertex_first,vertex_last timeout 1500 python tools/order_sweep.py w25,w26,w27 > gpurun_out/r2as_order_sweep.jsonl 2>&1; cut -c1-200 gpurun_out/r2as_order_sweep.jsonl
