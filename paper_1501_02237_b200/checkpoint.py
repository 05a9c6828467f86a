"""Checkpoint / resume of a long enumeration: the rank space
[0, C(N,K)) is a 1-D integer interval, so a checkpoint is the set of finished
contiguous rank intervals plus the running exact sums.  Each interval is one
bdeg_degree_range call (the kernel does all the work); this module only keeps
the ledger on disk, so a killed job restarts where it stopped."""
from __future__ import annotations

import json
import math
import os

from .bdeg import BDEG_E_DEGENERATE, BDEG_E_INVALID, BdegError, Plan

KEYS = ("degree", "cells", "singular", "candidates", "ties")


def degree_checkpointed(plan: Plan, path: str, chunks: int = 64, stop_after: int | None = None) -> dict:
    """The whole rank space in `chunks` contiguous colex-rank intervals, the
    running sums written to `path` (JSON, atomically) after each interval.
    A rerun with a plan of the same configuration and lifting resumes from the
    ledger.  `stop_after` (tests) stops after that many new intervals.
    Returns the sums; raises BDEG_E_DEGENERATE if the lifting had ties."""
    K, V, w = plan.points()
    total = math.comb(len(V), K)
    ident = {"K": K, "N": len(V), "total": total, "chunks": chunks,
             "seed_used": plan.info().seed_used, "lifting_hash": hash(tuple(w)) & ((1 << 61) - 1)}
    state = {"ident": ident, "done": [], "sums": {k: 0 for k in KEYS}}
    if os.path.exists(path):
        with open(path) as f:
            old = json.load(f)
        if old.get("ident") != ident:
            raise BdegError(BDEG_E_INVALID, f"checkpoint {path} belongs to another configuration or lifting")
        state = old
    done = set(state["done"])
    step = -(-total // chunks)
    new = 0
    for i in range(chunks):
        if i in done:
            continue
        if stop_after is not None and new >= stop_after:
            return state["sums"]
        b, e = i * step, min(total, (i + 1) * step)
        r = plan.degree_range(b, e) if b < e else None
        if r is not None:
            for k, v in (("degree", r.degree), ("cells", r.cells), ("singular", r.singular),
                         ("candidates", r.candidates), ("ties", r.ties)):
                state["sums"][k] += v
        state["done"].append(i)
        tmp = path + ".tmp"
        with open(tmp, "w") as f:
            json.dump(state, f)
        os.replace(tmp, path)
        new += 1
    if state["sums"]["ties"]:
        raise BdegError(BDEG_E_DEGENERATE, "degenerate lifting: re-lift (bdeg_relift) and start a new ledger")
    return state["sums"]
