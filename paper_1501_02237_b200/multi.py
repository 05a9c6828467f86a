"""Multi-GPU combine (one process per GPU, torch.distributed as plumbing).

Each rank runs bdeg_degree_partial over its share of the work items into a
16-slot int64 device buffer; one all-reduce(SUM) over NCCL (NVLink/NVSwitch)
combines them; bdeg_finalize carry-normalises the four 32-bit volume limbs
into the exact 128-bit degree (include/bdeg.h).

Degeneracy ("almost all" liftings): the tie count travels
in the same all-reduce.  Every rank sees the same summed slots, so every rank
takes the same decision: a generated lifting is re-drawn on all ranks with the
same attempt number (bdeg_relift, a deterministic derived seed) and the step
is recomputed; a user lifting raises BDEG_E_DEGENERATE everywhere.
"""
from __future__ import annotations

from .bdeg import BDEG_E_DEGENERATE, BDEG_E_INVALID, NSLOTS, BdegError, Plan, Result

MASK32 = (1 << 32) - 1
SLOT_TIES = 7


def pack_slots(volume: int, cells: int, singular: int, candidates: int, ties: int = 0,
               items: int = 0, updates: int = 0, leaves: int = 0):
    """Host-side slot layout of include/bdeg.h (for CPU ranks and tests)."""
    s = [0] * NSLOTS
    for i in range(4):
        s[i] = (volume >> (32 * i)) & MASK32
    s[4], s[5], s[6], s[7] = cells, singular, candidates, ties
    s[11], s[12], s[13] = items, updates, leaves
    return s


def all_reduce_slots(slots, group=None):
    import torch.distributed as dist
    dist.all_reduce(slots, op=dist.ReduceOp.SUM, group=group)
    return slots


def enable_work_stealing(plan: Plan, device: int, group=None):
    """All ranks draw the tail of the work items from one queue in rank 0's GPU
    memory (CUDA IPC + system-scope atomics over NVLink) after their static
    interleaved share (bdeg_steal_attach)."""
    import torch.distributed as dist
    from .bdeg import steal_create
    obj = [steal_create(device) if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    plan.steal_attach(obj[0])     # rank 0 resolves its own handle locally


def combine_with_relift(plan: Plan, partial, reduce, max_relift: int = 32) -> Result:
    """The collective degree protocol, independent of where the shard runs.

    partial(plan) -> this rank's 16 slots (any object `reduce` accepts);
    reduce(slots) -> the slots summed over all ranks, as a list of ints.
    Repeats with bdeg_relift(attempt + 1) on every rank while the summed tie
    count is non-zero (identical on all ranks, so all ranks agree)."""
    attempt = plan.info().relifts
    while True:
        summed = reduce(partial(plan))
        try:
            return plan.finalize(summed)
        except BdegError as e:
            if e.status != BDEG_E_DEGENERATE or summed[SLOT_TIES] == 0:
                raise
            if attempt + 1 > max_relift:
                raise BdegError(BDEG_E_DEGENERATE,
                                f"no generic lifting within {max_relift} re-lifts") from e
            try:
                plan.relift(attempt + 1)
            except BdegError as e2:       # a user lifting is never changed silently
                if e2.status == BDEG_E_INVALID:
                    raise e from None
                raise
            attempt += 1


def degree_distributed(plan: Plan, device, group=None, max_relift: int = 32) -> Result:
    """This rank's shard on `device`, one all-reduce per attempt, exact
    finalize, collective re-lift on a degenerate generated lifting."""
    import torch

    def partial(p):
        slots = torch.zeros(NSLOTS, dtype=torch.int64, device=device)
        p.degree_partial(slots.data_ptr())
        return slots

    def reduce(slots):
        all_reduce_slots(slots, group)
        return slots.cpu().tolist()

    return combine_with_relift(plan, partial, reduce, max_relift)


class _CudaBuf:
    """A raw device pointer seen by torch without a copy (__cuda_array_interface__)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 2, "strides": None}


def degree_walk_distributed(plan: Plan, group=None) -> Result:
    """the cell walk with its hash set sharded over the ranks of
    `group` (owner = hash(cell) mod world; one all-to-all of the neighbours
    owned elsewhere per level; the volumes summed by one all-reduce).  NCCL:
    the cells move device to device; gloo (tests): staged through the host."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device())

    def allreduce_sum(vals):
        t = torch.tensor(vals, dtype=torch.int64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t.cpu().tolist()

    def alltoall_counts(send):
        t = torch.tensor(send, dtype=torch.int64, device=dev if backend == "nccl" else "cpu")
        out = torch.empty_like(t)
        dist.all_to_all_single(out, t, group=group)
        return out.cpu().tolist()

    def alltoall_cells(d_send, scnt, d_recv, rcnt):
        ns, nr = 16 * sum(scnt), 16 * sum(rcnt)
        send = torch.as_tensor(_CudaBuf(d_send, ns), device=dev) if ns else torch.empty(0, dtype=torch.uint8, device=dev)
        recv = torch.as_tensor(_CudaBuf(d_recv, nr), device=dev) if nr else torch.empty(0, dtype=torch.uint8, device=dev)
        if backend == "nccl":
            dist.all_to_all_single(recv, send, output_split_sizes=[16 * c for c in rcnt],
                                   input_split_sizes=[16 * c for c in scnt], group=group)
            torch.cuda.current_stream().synchronize()
        else:
            hr = torch.empty(nr, dtype=torch.uint8)
            dist.all_to_all_single(hr, send.cpu(), output_split_sizes=[16 * c for c in rcnt],
                                   input_split_sizes=[16 * c for c in scnt], group=group)
            if nr:
                recv.copy_(hr)
            torch.cuda.current_stream().synchronize()

    return plan.degree_walk_sharded(allreduce_sum, alltoall_counts, alltoall_cells)
