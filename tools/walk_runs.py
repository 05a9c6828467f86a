#!/usr/bin/env python
"""Degree by the cell walk (bdeg_degree_walk) on bench workloads; one JSON line each."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1501_02237_b200 as B  # noqa: E402

torch.cuda.set_device(0)
for wl in sys.argv[1].split(","):
    if wl.startswith("w"):   # the binomial system itself, generated lifting (basis-seeded if N > 64)
        import workloads as W
        A, b = W.master_space_system(int(wl[1]), int(wl[2]))
        p = B.Plan.from_system(A, b, seed=int(os.environ.get("WALK_SEED", "1")))
    else:
        p = bench.Workload(wl).plan()
    K, nv = p.info().K, p.info().N
    t0 = time.perf_counter()
    r = p.degree_walk()
    dt = time.perf_counter() - t0
    print(json.dumps({"wl": wl, "seed": int(os.environ.get("WALK_SEED", "1")), "K": K, "N": nv, "candidates": math.comb(nv, K), "walk_s": dt,
                      "kernel_ms": r.kernel_ms, "degree": r.degree, "cells": r.cells,
                      "ridge_tests": r.leaves, "boundary_ridges": r.dead_leaves,
                      "simplices_per_s": math.comb(nv, K) / dt}), flush=True)
    p.close()
