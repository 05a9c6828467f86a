#!/bin/bash
# round 2, call AQ: point-order sweep, more workloads (W34, W27 full; W35, W44 degree-only)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SWEEP_ORDERS=planner,reversed,lift_asc,norm_desc timeout 1200 python tools/order_sweep.py w34,w24,w27 > gpurun_out/r2aq_order_sweep.jsonl 2>&1
SWEEP_FLAGS=0x40 SWEEP_ORDERS=planner,reversed,lift_asc,norm_desc timeout 1500 python tools/order_sweep.py w35,w44 >> gpurun_out/r2aq_order_sweep.jsonl 2>&1
cut -c1-200 gpurun_out/r2aq_order_sweep.jsonl
