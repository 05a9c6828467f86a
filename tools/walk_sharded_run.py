#!/usr/bin/env python
"""Sharded cell walk (bdeg_degree_walk_sharded) with W ranks sharing the visible GPU(s) over gloo,
against the one-rank walk: `python tools/walk_sharded_run.py w45 [world]`; one JSON line each."""
import json
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, wl, q):
    import torch
    import torch.distributed as dist
    import workloads as W
    import paper_1501_02237_b200 as B
    from paper_1501_02237_b200.multi import degree_walk_distributed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A, b = W.master_space_system(int(wl[1]), int(wl[2]))
    plan = B.Plan.from_system(A, b, seed=1, rank=rank, world=world, device=rank % torch.cuda.device_count())
    dist.barrier()
    t0 = time.perf_counter()
    r = degree_walk_distributed(plan)
    q.put((rank, r.degree, r.cells, time.perf_counter() - t0))
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    import workloads as W
    import paper_1501_02237_b200 as B
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    for wl in sys.argv[1].split(","):
        A, b = W.master_space_system(int(wl[1]), int(wl[2]))
        t0 = time.perf_counter()
        one = B.Plan.from_system(A, b, seed=1).degree_walk()
        t1 = time.perf_counter() - t0
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _port()
        ps = [ctx.Process(target=_worker, args=(r, world, port, wl, q)) for r in range(world)]
        for p in ps:
            p.start()
        res = sorted(q.get(timeout=3600) for _ in ps)
        for p in ps:
            p.join()
        print(json.dumps({"wl": wl, "world": world, "one_rank": {"degree": one.degree, "cells": one.cells, "s": t1},
                          "sharded": [{"rank": r, "degree": d, "cells": c, "s": s} for r, d, c, s in res],
                          "equal": all(d == one.degree and c == one.cells for _, d, c, _ in res)}), flush=True)
