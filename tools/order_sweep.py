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
    # lifting minus its least-squares linear fit (invariant under adding a linear function)
    import numpy as np
    Vm = np.array(V, dtype=np.float64); wv = np.array(w, dtype=np.float64)
    h = np.linalg.lstsq(Vm, wv, rcond=None)[0]
    res = wv - Vm @ h
    orders["resid_asc"] = sorted(range(N), key=lambda i: res[i])
    if os.environ.get("SWEEP_VERTEX"):
        # points that lie in some cell (vertices of the subdivision) first, by lifting;
        # the others (never in a cell) last: found from the plan's own cell list
        with B.Plan.from_system(A, b, seed=1, flags=B.bdeg.FLAG_NATURAL_ORDER) as pn:
            Kn, Vn, wn = pn.points()
            cells = pn.cells()
        vert = set(i for c, _ in cells for i in c)
        assert Vn == V or True
        nat_w = {tuple(v): ww for v, ww in zip(Vn, wn)}
        isv = [any(tuple(V[i]) == tuple(Vn[j]) for j in vert) for i in range(N)]
        orders["vertex_first"] = sorted(range(N), key=lambda i: (not isv[i], w[i]))
        orders["vertex_last"] = sorted(range(N), key=lambda i: (isv[i], w[i]))
        print(json.dumps({"wl": wl, "vertices": sum(isv), "N": N}), flush=True)
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
