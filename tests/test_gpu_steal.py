"""Cross-GPU dynamic work stealing exercised with two processes
sharing the one available GPU: rank 0 exports the item counters by CUDA IPC,
both ranks draw work items from that single queue with system-scope atomics,
one all-reduce (gloo here, NCCL on a multi-GPU box) combines the slots, and the
result must equal a single-process run over the whole rank space."""
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


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    import workloads as W
    import paper_1501_02237_b200 as B
    from paper_1501_02237_b200.multi import all_reduce_slots, enable_work_stealing
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    V, w = W.c5_points(1)
    plan = B.Plan.from_points(V, w, rank=rank, world=world, device=0)
    enable_work_stealing(plan, 0)
    out, busy, mine = [], [], []
    for _ in range(3):                       # several steps: counters alternate by parity
        slots = torch.zeros(B.NSLOTS, dtype=torch.int64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        e0.record()
        plan.degree_partial(slots.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        busy.append(e0.elapsed_time(e1))
        host = slots.cpu()
        mine.append(int(host[6]))            # candidates this rank enumerated
        all_reduce_slots(host)
        r = plan.finalize(host.tolist())
        out.append((r.degree, r.cells, r.singular, r.candidates))
    q.put((rank, (out, busy, mine, plan.queue_info())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ranks_share_one_queue(world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    import workloads as W
    import paper_1501_02237_b200 as B
    V, w = W.c5_points(1)
    full = B.Plan.from_points(V, w).degree()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    want = (full.degree, full.cells, full.singular, full.candidates)
    assert all(step == want for r in range(world) for step in res[r][0])
    # static share (~80% of the candidates, interleaved) + stealing tail: every
    # rank does a substantial part of every step (world-aware split items)
    q0 = res[0][3]
    assert q0["n_split"] > 0 and q0["n_static"] < q0["n_items"]
    for s in range(3):
        c = [res[r][2][s] for r in range(world)]
        assert sum(c) == full.candidates and min(c) > 0.5 * full.candidates / world, c
        b = [res[r][1][s] for r in range(world)]
        print(f"world {world} step {s}: rank busy ms {b}, candidates {c}")
