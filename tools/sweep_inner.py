#!/usr/bin/env python
"""Sweep the register-DFS depth S (inner_levels) on a few workloads; prints ms and rate."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1501_02237_b200 as B  # noqa: E402

wls = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c5", "w25", "w26"]
Ss = [int(s) for s in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 3, 4, 5, 6]
torch.cuda.set_device(0)
for wl in wls:
    W = bench.Workload(wl)          # the library's own front end (bdeg_plan / bdeg_plan_points)
    for S in Ss:
        p = W.plan(inner_levels=S, flags=int(os.environ.get("SWEEP_FLAGS", "0"), 0))
        info = p.info()
        if S > info.K - 1:
            p.close()
            continue
        total = math.comb(info.N, info.K)
        r = p.degree()   # warm
        reps = 3 if total < 1e10 else 1
        t0 = time.perf_counter()
        for _ in range(reps):
            r = p.degree()
        dt = (time.perf_counter() - t0) / reps
        print(json.dumps({"wl": wl, "S": S, "tier": r.tier, "ms": dt * 1e3, "kernel_ms": r.kernel_ms,
                          "rate": total / dt, "degree": r.degree, "leaves": r.leaves, "dead": r.dead_leaves}), flush=True)
        p.close()
