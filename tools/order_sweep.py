#!/usr/bin/env python
"""Point-order sweep (reading O: the order changes ranks and work, never results): the
configuration the planner builds from x^A = b, enumerated under several orders."""
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_1501_02237_b200 as B  # noqa: E402

torch.cuda.set_device(0)
flags = int(os.environ.get("SWEEP_FLAGS", "0"), 0)           # 0x40: degree-only
only = os.environ.get("SWEEP_ORDERS")
for wl in sys.argv[1].split(","):
    m, k = int(wl[1]), int(wl[2])
    A, b = W.master_space_system(m, k)
    with B.Plan.from_system(A, b, seed=1, flags=flags) as p:
        K, V, w = p.points()
        base = p.degree()
    N = len(V)
    norms = [sum(x * x for x in v) for v in V]
    orders = {"planner": list(range(N)), "reversed": list(range(N))[::-1],
              "lift_asc": sorted(range(N), key=lambda i: w[i]), "lift_desc": sorted(range(N), key=lambda i: -w[i]),
              "norm_asc": sorted(range(N), key=lambda i: norms[i]), "norm_desc": sorted(range(N), key=lambda i: -norms[i])}
    for s in range(3):
        o = list(range(N)); random.Random(s).shuffle(o); orders[f"random{s}"] = o
    for name, o in orders.items():
        if only and name not in only.split(","):
            continue
        Vo, wo = [V[i] for i in o], [w[i] for i in o]
        with B.Plan.from_points(Vo, wo, flags=flags) as q:
            r = q.degree()
            if r.kernel_ms < 2000:
                r = q.degree()
        assert (r.degree, r.cells) == (base.degree, base.cells)
        assert flags or r.singular == base.singular
        print(json.dumps({"wl": wl, "order": name, "K": K, "N": N, "kernel_ms": r.kernel_ms, "leaves": r.leaves,
                          "dead": r.dead_leaves, "dead_full": r.dead_full}), flush=True)
