#!/bin/bash
# round 2, call AZ: lifting order vs the order of the lifting's residual after its least-squares linear fit
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SWEEP_ORDERS=planner,resid_asc timeout 1200 python tools/order_sweep.py w25,w26,w34,w27 > gpurun_out/r2az_order_sweep.jsonl 2>&1
SWEEP_FLAGS=0x40 SWEEP_ORDERS=planner,resid_asc timeout 1200 python tools/order_sweep.py w35 >> gpurun_out/r2az_order_sweep.jsonl 2>&1
cut -c1-160 gpurun_out/r2az_order_sweep.jsonl
