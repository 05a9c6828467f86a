"""ctypes wrapper of oracle/c/bdeg_oracle.c — test infrastructure only.

An interval on which __int128 overflows (status 1) is recomputed with the
Python Fraction oracle (exact, slow); `fallback` counts such intervals.

The C file is the brute force of oracle/subdivision.py (cone test, Cramer's
rule in checked __int128); it is compiled by __graft_entry__.build() (or on
first use here) with plain gcc into oracle/c/libbdeg_oracle.so.  Rank
intervals are split across host threads (ctypes releases the GIL), which is
how bench.py times the oracle on the box's host cores.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "c", "bdeg_oracle.c")
_LIB = os.path.join(_HERE, "c", "libbdeg_oracle.so")
_lock = threading.Lock()
_lib = None


def build_oracle_lib(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build_oracle_lib()
            lib = ctypes.CDLL(_LIB)
            lib.bdeg_oracle_enumerate.argtypes = [
                ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                ctypes.POINTER(ctypes.c_int64), ctypes.c_uint64, ctypes.c_uint64,
                ctypes.POINTER(ctypes.c_int64)]
            lib.bdeg_oracle_enumerate.restype = ctypes.c_int
            _lib = lib
    return _lib


def _one(K, N, Vbuf, wbuf, b, e, V=None, lifts=None):
    out = (ctypes.c_int64 * 7)()
    _load().bdeg_oracle_enumerate(K, N, Vbuf, wbuf, b, e, out)
    if out[6] == 1 and V is not None:
        # __int128 overflowed: redo this interval with Python's exact ints
        from .subdivision import enumerate_lifted
        r = enumerate_lifted(K, V, lifts, b, e, "cone")
        r["status"] = 0
        r["fallback"] = 1
        return r
    vol = (out[1] & ((1 << 64) - 1)) << 64 | (out[0] & ((1 << 64) - 1))
    if out[1] < 0:
        vol -= 1 << 128
    return {"volume": vol, "cells": out[2], "singular": out[3],
            "candidates": out[4], "ties": out[5], "status": out[6]}


def enumerate_range(K, V, lifts, rank_begin=0, rank_end=None, threads=1, chunk=None):
    """Counts over colex ranks [rank_begin, rank_end) of K-subsets of the
    K-vectors V (point-major) with lifts.  Same semantics as
    oracle.subdivision.enumerate_lifted(test="cone")."""
    from .subdivision import binom
    N = len(V)
    total = binom(N, K)
    if rank_end is None or rank_end > total:
        rank_end = total
    Vbuf = (ctypes.c_int64 * (N * K))(*[int(x) for v in V for x in v])
    wbuf = (ctypes.c_int64 * N)(*[int(x) for x in lifts])
    span = max(0, rank_end - rank_begin)
    if chunk is None:
        chunk = max(1, -(-span // max(1, threads * 8)))
    pieces = [(b, min(b + chunk, rank_end)) for b in range(rank_begin, rank_end, chunk)]
    res = {"volume": 0, "cells": 0, "singular": 0, "candidates": 0, "ties": 0, "status": 0}
    if not pieces:
        return res
    if threads <= 1:
        parts = [_one(K, N, Vbuf, wbuf, b, e, V, lifts) for b, e in pieces]
    else:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            parts = list(ex.map(lambda be: _one(K, N, Vbuf, wbuf, be[0], be[1], V, lifts), pieces))
    for p in parts:
        res["fallback"] = res.get("fallback", 0) + p.get("fallback", 0)
        for k in ("volume", "cells", "singular", "candidates", "ties", "status"):
            if k == "status":
                res[k] = max(res[k], p[k])
            else:
                res[k] += p[k]
    return res
