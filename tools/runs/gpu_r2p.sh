#!/bin/bash
# Table 3 enumeration runs through the library front end (round-2 kernel)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python - > gpurun_out/r2p_table3_enum.jsonl 2>&1 <<'PY'
import json, math, sys, time
sys.path.insert(0, ".")
import torch, workloads as W, paper_1501_02237_b200 as B
torch.cuda.set_device(0)
for (m, k, flags) in [(2, 7, 0), (2, 7, B.bdeg.FLAG_DEGREE_ONLY), (3, 5, B.bdeg.FLAG_DEGREE_ONLY),
                      (4, 4, B.bdeg.FLAG_DEGREE_ONLY), (2, 8, B.bdeg.FLAG_DEGREE_ONLY)]:
    A, b = W.master_space_system(m, k)
    t0 = time.perf_counter()
    with B.Plan.from_system(A, b, seed=1, flags=flags) as p:
        r = p.degree()
    dt = time.perf_counter() - t0
    tot = math.comb(r.N, r.K)
    print(json.dumps({"m": m, "k": k, "mode": "degree-only" if flags else "full", "K": r.K, "N": r.N,
                      "candidates": tot, "degree": r.degree, "cells": r.cells, "singular": r.singular,
                      "singular_complete": r.singular_complete, "kernel_s": r.kernel_ms / 1e3, "wall_s": dt,
                      "simplices_per_s": tot / (r.kernel_ms / 1e3), "dead_full": r.dead_full}), flush=True)
PY
cat gpurun_out/r2p_table3_enum.jsonl | cut -c1-300
