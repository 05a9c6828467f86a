#!/usr/bin/env python
"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): `compute-sanitizer --tool racecheck python tools/sanitize_run.py`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
import paper_1501_02237_b200 as B  # noqa: E402

V, w = W.c5_points(1, n_points=20, dim=4)
p = B.Plan.from_points(V, w)
r = p.degree()                                        # k_enumerate (tier 1) + replays
print("enumerate", r.degree, r.cells)
print("range", p.degree_range(100, 9000).degree)      # mode-0 items
print("cells", len(p.cells()))
print("walk", p.degree_walk().degree)                 # start search + k_walk_dc
V2, w2 = W.c5_points(1, n_points=40, dim=4)           # N > 32: both point slots of the leaf
print("enumerate N=40", B.Plan.from_points(V2, w2).degree().degree)
A, b = W.master_space_system(2, 3)
print("W23", B.degree(A, b).degree, B.Plan.from_system(A, b).degree_walk().degree)
rng = W.SplitMix64(1)
Vw = [(1,) + tuple(rng.uniform_int(-(1 << 30), 1 << 30) for _ in range(2)) for _ in range(9)]
ww = [rng.next() >> 14 for _ in range(9)]
r = B.Plan.from_points(Vw, ww).degree()                # tier 2 -> tier 4 (int128 values)
print("wide", r.degree, r.wide_reruns)
A, b = W.master_space_system(4, 4)
An = np.array(A, dtype=np.int64)
print("smith", B.smith_gpu(An), "dim_modp", B.dimension_modp(An))
