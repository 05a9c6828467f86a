"""the cell walk with its hash set sharded over the ranks
(owner = hash(cell) mod world, one all-to-all of the neighbours per level, the
volumes summed by one all-reduce) — the paper's shared KnownNodes table
 rebuilt owner-computes.  Two processes share the one GPU of the
box and exchange over gloo; the result must equal the single-process walk
(same lifting => same subdivision) and Table 3."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cases():
    import workloads as W
    out = []
    A, b = W.master_space_system(3, 6)                     # Table 3: 7029180, N = 54
    out.append(("W36", ("system", A, b, None, 1)))
    A, b = W.master_space_system(2, 5)
    out.append(("W25", ("system", A, b, None, 1)))
    V, _ = W.c5_points(5, n_points=80, dim=3, lo=-4, hi=4)  # N > 64: basis-seeded start cell
    out.append(("pts80", ("points", V, None, None, 5)))
    A, b = W.master_space_system(2, 2)                      # 2-bit liftings: a collective re-lift
    out.append(("W22relift", ("system", A, b, 2, 3)))
    return out


def _plan(case, **opts):
    import paper_1501_02237_b200 as B
    kind, X, b, bits, seed = case
    extra = {"lift_bits": bits} if bits else {}
    if kind == "system":
        return B.Plan.from_system(X, b, seed=seed, **extra, **opts)
    return B.Plan.from_points(X, None, seed=seed, **extra, **opts)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["BDEG_DEBUG"] = "1"
    import torch.distributed as dist
    from paper_1501_02237_b200.multi import degree_walk_distributed
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    for name, case in _cases():
        plan = _plan(case, rank=rank, world=world, device=0)
        r = degree_walk_distributed(plan)
        out[name] = (r.degree, r.cells, r.relifts)
    q.put((rank, out))
    dist.destroy_process_group()


def test_sharded_walk_two_ranks_equals_single(capfd):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    single = {}
    for name, case in _cases():
        r = _plan(case, device=0).degree_walk()
        single[name] = (r.degree, r.cells, r.relifts)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    err = capfd.readouterr().err
    assert res[0] == res[1] == single, (res, single)
    assert single["W36"][0] == 7029180 and single["W25"][0] == 3632 and single["W22relift"][0] == 14
    assert single["W22relift"][2] >= 1
    # both ranks owned and exchanged cells
    lines = [l for l in err.splitlines() if "sharded walk] rank" in l]
    owned = [int(l.split(" owned cells")[0].split(", ")[-1]) for l in lines]
    assert len(lines) >= 2 and min(owned) > 0, err[-3000:]
