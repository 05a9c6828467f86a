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
    desc, K, V, w, extra = bench.workload(wl)
    p = B.Plan.from_points(V, w)
    t0 = time.perf_counter()
    r = p.degree_walk()
    dt = time.perf_counter() - t0
    print(json.dumps({"wl": wl, "K": K, "N": len(V), "candidates": math.comb(len(V), K), "walk_s": dt,
                      "kernel_ms": r.kernel_ms, "degree": r.degree, "cells": r.cells,
                      "ridge_tests": r.leaves, "boundary_ridges": r.dead_leaves,
                      "simplices_per_s": math.comb(len(V), K) / dt}), flush=True)
    p.close()
