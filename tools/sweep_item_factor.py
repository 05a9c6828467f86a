"""Device time of bdeg_degree on C5 for several work-item granularities
(BDEG_ITEM_FACTOR, read by the planner).  Usage on a GPU box:
    python tools/sweep_item_factor.py 0.125 0.25 0.5 1"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
import paper_1501_02237_b200 as B  # noqa: E402

V, w = W.c5_points(1)
for f in sys.argv[1:]:
    os.environ["BDEG_ITEM_FACTOR"] = f
    with B.Plan.from_points(V, w) as p:
        ms = []
        for i in range(23):
            r = p.degree()
            if i >= 3:
                ms.append(r.kernel_ms)
        print(f"factor {f}: items {p.num_items()} kernel_ms median {statistics.median(ms):.3f} "
              f"min {min(ms):.3f} degree {r.degree}", flush=True)
