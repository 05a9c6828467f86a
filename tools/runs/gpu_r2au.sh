#!/bin/bash
# round 2, call AU: does the lifting order help the C5 point configuration (caller's order kept by bdeg_plan_points)?
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python - > gpurun_out/r2au_c5_order.jsonl 2>&1 <<'PY'
import json, sys
sys.path.insert(0, ".")
import torch, workloads as W, paper_1501_02237_b200 as B
torch.cuda.set_device(0)
V, w = W.c5_points(1)
N = len(V)
orders = {"caller": list(range(N)), "lift_asc": sorted(range(N), key=lambda i: w[i]),
          "lift_desc": sorted(range(N), key=lambda i: -w[i]), "reversed": list(range(N))[::-1]}
for name, o in orders.items():
    with B.Plan.from_points([V[i] for i in o], [w[i] for i in o]) as p:
        ms = []
        for _ in range(7):
            r = p.degree(); ms.append(r.kernel_ms)
    print(json.dumps({"order": name, "kernel_ms_min": min(ms[2:]), "degree": r.degree, "leaves": r.leaves}), flush=True)
PY
cat gpurun_out/r2au_c5_order.jsonl
