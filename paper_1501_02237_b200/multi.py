"""Multi-GPU combine (one process per GPU, torch.distributed as plumbing).

Each rank runs bdeg_degree_partial over its interleaved share of the work
items into a 16-slot int64 device buffer; one all-reduce(SUM) over NCCL
(NVLink/NVSwitch) combines them; bdeg_finalize carry-normalises the four
32-bit volume limbs into the exact 128-bit degree (include/bdeg.h).
"""
from __future__ import annotations

from .bdeg import NSLOTS, Plan, Result

MASK32 = (1 << 32) - 1


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
    """All ranks draw work items from one queue in rank 0's GPU memory (CUDA
    IPC + system-scope atomics over NVLink), instead of static shards."""
    import torch.distributed as dist
    from .bdeg import steal_create
    obj = [steal_create(device) if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    plan.steal_attach(obj[0])     # rank 0 resolves its own handle locally


def degree_distributed(plan: Plan, device, group=None) -> Result:
    """This rank's shard on `device`, one all-reduce, exact finalize."""
    import torch
    slots = torch.zeros(NSLOTS, dtype=torch.int64, device=device)
    plan.degree_partial(slots.data_ptr())
    all_reduce_slots(slots, group)
    return plan.finalize(slots.cpu().tolist())
