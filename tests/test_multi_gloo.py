"""World-size-2 test of the multi-GPU path on CPU (gloo): each rank plans the
same problem deterministically, computes its interleaved share of the work
items (here with the CPU oracle standing in for the GPU kernel), packs the
16 result slots, one all-reduce(SUM) combines them, and bdeg_finalize (the
C ABI's host-side combine) must give the full-rank-space result."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1501_02237_b200 as B
    from paper_1501_02237_b200.multi import all_reduce_slots, pack_slots
    from oracle.native import enumerate_range
    out = []
    for (V, w, K) in cases:
        plan = B.Plan.from_points(V, w, rank=rank, world=world)
        # the plan is replicated: every rank must see the same decomposition
        n = torch.tensor([plan.num_items()], dtype=torch.int64)
        mx = n.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        assert int(mx) == int(n)
        acc = {"volume": 0, "cells": 0, "singular": 0, "candidates": 0, "ties": 0}
        for it in plan.shard_items(rank, world):
            b, e = plan.item_range(it)
            r = enumerate_range(K, V, w, b, e)
            for k in acc:
                acc[k] += r[k]
        slots = torch.tensor(pack_slots(acc["volume"], acc["cells"], acc["singular"],
                                        acc["candidates"], acc["ties"]), dtype=torch.int64)
        all_reduce_slots(slots)
        res = plan.finalize(slots.tolist())
        out.append((res.degree, res.cells, res.singular, res.candidates))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_combine_gloo(world):
    cases = []
    V, w = W.c5_points(3, n_points=14, dim=4)
    cases.append((V, w, 5))
    from oracle import point_configuration
    A, b = W.master_space_system(2, 2)
    K, V2, w2 = point_configuration(A, b, W.liftings(len(A) + 1, 1))["cone"]
    cases.append((V2, w2, K))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    from oracle.native import enumerate_range
    for i, (V, w, K) in enumerate(cases):
        full = enumerate_range(K, V, w)
        want = (full["volume"], full["cells"], full["singular"], full["candidates"])
        assert res[0][i] == res[1][i] == want
    assert res[0][1][0] == 14          # W_{2,2}: Table 3


def _relift_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1501_02237_b200 as B
    from paper_1501_02237_b200.multi import all_reduce_slots, combine_with_relift, pack_slots
    from oracle.native import enumerate_range
    # 2-bit generated liftings of W_{2,2}: degenerate at attempt 0
    A, b = W.master_space_system(2, 2)
    plan = B.Plan.from_system(A, b, seed=3, lift_bits=2, rank=rank, world=world)
    attempts = []

    def partial(p):
        K, V, w = p.points()                 # the lifting in use on this attempt
        attempts.append(p.info().seed_used)
        acc = {"volume": 0, "cells": 0, "singular": 0, "candidates": 0, "ties": 0}
        for it in p.shard_items(rank, world):
            bb, e = p.item_range(it)
            r = enumerate_range(K, V, w, bb, e)
            for k in acc:
                acc[k] += r[k]
        return torch.tensor(pack_slots(acc["volume"], acc["cells"], acc["singular"],
                                       acc["candidates"], acc["ties"]), dtype=torch.int64)

    def reduce(slots):
        all_reduce_slots(slots)
        return slots.tolist()

    res = combine_with_relift(plan, partial, reduce)
    # a user lifting with ties is never re-lifted: every rank raises
    K, V, w = plan.points()
    flat = [7] * (len(A) + 1)
    plan2 = B.Plan.from_system(A, b, flat, rank=rank, world=world)
    try:
        combine_with_relift(plan2, partial, reduce)
        raised = None
    except B.BdegError as e:
        raised = e.status
    q.put((rank, (res.degree, res.relifts, res.seed_used, tuple(attempts[:res.relifts + 1]), raised)))
    dist.destroy_process_group()


def test_collective_relift_gloo():
    """Ties travel in the all-reduce; every rank re-lifts with the same attempt
    (SURVEY §8.e degeneracy row) and the combined degree is exact."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_relift_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0][:4] == res[1][:4]
    deg, relifts, seed, seeds, raised = res[0]
    assert deg == 14 and relifts >= 1          # W_{2,2}: Table 3
    assert len(set(seeds)) == relifts + 1      # a fresh lifting per attempt
    assert raised == 3 and res[1][4] == 3      # BDEG_E_DEGENERATE on every rank
