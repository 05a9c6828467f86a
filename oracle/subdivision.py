"""Degree as the volume of a regular simplicial subdivision — PAPER.md §4,
P:665-800, by the brute force the paper names at P:798-800.

Test infrastructure only (see oracle/__init__.py).

For a lifting omega: S -> R the projections of the d-dimensional
lower faces of conv(S^) form a simplicial subdivision for almost all omega
(P:727-730); the degree is the sum of the normalised volumes of its cells
(P:687-697).  A set {a_0..a_d} spans a lower d-face iff the system
I(a_0..a_d) (eq. lower-face) is feasible:

    <a^_0, alpha^> = <a^_j, alpha^>   j = 1..d
    <a^_0, alpha^> <= <a^, alpha^>    a in S,      alpha^ = (alpha, 1).

Readings:
  Z1  NVol(conv{a_0..a_d}) = |det(a_1-a_0, ..., a_d-a_0)| (eq. simplex-vol,
      P:690-695, is garbled: a d x (d+1) "determinant").
  Z3  The inequality is taken strictly for a not in the cell; a candidate
      with no strictly violated inequality but some equality (a tie) means
      the lifting is not generic ("almost all") -> `ties` is counted
      and the caller must re-lift.  A zero for a rejected candidate is benign.

Enumeration order: K-subsets c_0 < c_1 < ... < c_{K-1} of {0..N-1} in
co-lexicographic order, rank = sum_i C(c_i, i+1) (combinatorial number
system).  `rank_begin/rank_end` restrict to a rank interval.

All arithmetic is exact (Python ints and fractions.Fraction).
"""
from __future__ import annotations

from fractions import Fraction
from math import comb

from .points import point_configuration


def binom(n: int, k: int) -> int:
    return comb(n, k) if 0 <= k <= n else 0


def colex_rank(c) -> int:
    """rank of the sorted tuple c (combinatorial number system)."""
    return sum(binom(ci, i + 1) for i, ci in enumerate(c))


def colex_unrank(r: int, K: int):
    """Inverse of colex_rank: greedy from the largest element down."""
    out = [0] * K
    for i in range(K - 1, -1, -1):
        c = i
        while binom(c + 1, i + 1) <= r:
            c += 1
        out[i] = c
        r -= binom(c, i + 1)
    return tuple(out)


def colex_next(c, N):
    """Successor of the sorted tuple c in colex order, or None."""
    c = list(c)
    K = len(c)
    for i in range(K):
        limit = c[i + 1] if i + 1 < K else N
        if c[i] + 1 < limit:
            c[i] += 1
            for t in range(i):
                c[t] = t
            return tuple(c)
    return None


def _solve(M, rhs):
    """Solve M x = rhs over Q (Gaussian elimination); M square, non-singular.
    Returns (det M, x)."""
    n = len(M)
    a = [[Fraction(v) for v in row] + [Fraction(r)] for row, r in zip(M, rhs)]
    det = Fraction(1)
    for c in range(n):
        p = next((i for i in range(c, n) if a[i][c] != 0), None)
        if p is None:
            return Fraction(0), None
        if p != c:
            a[c], a[p] = a[p], a[c]
            det = -det
        det *= a[c][c]
        for i in range(c + 1, n):
            if a[i][c] != 0:
                f = a[i][c] / a[c][c]
                a[i] = [x - f * y for x, y in zip(a[i], a[c])]
    x = [Fraction(0)] * n
    for i in range(n - 1, -1, -1):
        s = a[i][n] - sum(a[i][j] * x[j] for j in range(i + 1, n))
        x[i] = s / a[i][i]
    return det, x


def lower_face_affine(points, lifts, cell):
    """Paper-literal test of I(a_0..a_d) for the index tuple
    `cell` (d+1 indices into the affine points of S u {0}).

    Returns (status, nvol) with status in {"singular", "cell", "tie", "no"}.
    alpha solves <a_j - a_0, alpha> = omega(a_0) - omega(a_j), j = 1..d
    (the equalities of I with alpha^ = (alpha, 1))."""
    a0 = points[cell[0]]
    w0 = lifts[cell[0]]
    d = len(a0)
    M = [[points[cj][t] - a0[t] for t in range(d)] for cj in cell[1:]]
    rhs = [w0 - lifts[cj] for cj in cell[1:]]
    det, alpha = _solve(M, rhs)
    if det == 0:
        return "singular", 0
    nvol = abs(det)                       # Z1 reading of eq. simplex-vol
    assert nvol.denominator == 1
    base = sum(a0[t] * alpha[t] for t in range(d)) + w0   # <a^_0, alpha^>
    inside = set(cell)
    tie = False
    for i, a in enumerate(points):
        if i in inside:
            continue
        val = sum(a[t] * alpha[t] for t in range(d)) + lifts[i] - base
        if val < 0:
            return "no", int(nvol)        # a lifted point strictly below
        if val == 0:
            tie = True
    return ("tie" if tie else "cell"), int(nvol)


def lower_face_cone(V, lifts, sigma):
    """The same test in homogeneous coordinates: K vectors v_c (c in sigma)
    in Z^K.  h solves h . v_c = omega_c (c in sigma); sigma is a lower facet
    iff omega_l - h . v_l > 0 for every other l.  With V = (1, a) this is
    I(a_0..a_d) with h = (<a^_0, alpha^>, -alpha) (points.py docstring);
    with V = S in the homogeneous case it is the pyramid reading.
    NVol = |det V_sigma|."""
    K = len(sigma)
    M = [list(V[c]) for c in sigma]
    det, h = _solve(M, [lifts[c] for c in sigma])
    if det == 0:
        return "singular", 0
    inside = set(sigma)
    tie = False
    for l, v in enumerate(V):
        if l in inside:
            continue
        val = lifts[l] - sum(h[t] * v[t] for t in range(K))
        if val < 0:
            return "no", int(abs(det))
        if val == 0:
            tie = True
    return ("tie" if tie else "cell"), int(abs(det))


def enumerate_lifted(K, objs, lifts, rank_begin=0, rank_end=None, test="cone"):
    """Brute force over all K-subsets in colex rank order [rank_begin, rank_end)
    (P:798-800).  objs: cone vectors (test="cone") or affine points
    (test="affine").  Returns dict(volume, cells, singular, candidates, ties)."""
    N = len(objs)
    total = binom(N, K)
    if rank_end is None or rank_end > total:
        rank_end = total
    res = {"volume": 0, "cells": 0, "singular": 0, "candidates": 0, "ties": 0}
    if rank_begin >= rank_end:
        return res
    fn = lower_face_cone if test == "cone" else lower_face_affine
    c = colex_unrank(rank_begin, K)
    for _ in range(rank_end - rank_begin):
        status, nvol = fn(objs, lifts, c)
        res["candidates"] += 1
        if status == "singular":
            res["singular"] += 1
        elif status == "cell":
            res["cells"] += 1
            res["volume"] += nvol
        elif status == "tie":
            res["ties"] += 1
        c = colex_next(c, N)
    return res


def cell_list(K, objs, lifts, rank_begin=0, rank_end=None, test="cone"):
    """The cells themselves (index tuples with their NVol) among the ranks
    [rank_begin, rank_end) — the simplicial subdivision D of Def. 1."""
    N = len(objs)
    total = binom(N, K)
    if rank_end is None or rank_end > total:
        rank_end = total
    fn = lower_face_cone if test == "cone" else lower_face_affine
    out = []
    if rank_begin >= rank_end:
        return out
    c = colex_unrank(rank_begin, K)
    for _ in range(rank_end - rank_begin):
        status, nvol = fn(objs, lifts, c)
        if status == "cell":
            out.append((tuple(c), nvol))
        c = colex_next(c, N)
    return sorted(out)


def degree(A, b=None, lifting=None, test="cone", rank_begin=0, rank_end=None):
    """deg V of each component of V*(x^A - b) (Prop. 4) by the
    lifted brute force.  Returns dict(dim, components, degree, cells,
    singular, candidates, ties, K, N, homogeneous, consistent)."""
    cfg = point_configuration(A, b, lifting)
    out = {k: cfg[k] for k in ("dim", "components", "consistent", "homogeneous", "rank")}
    if not cfg["consistent"]:
        out["degree"] = None
        return out
    if cfg["dim"] == 0:                         # isolated points
        out.update(degree=1, cells=0, singular=0, candidates=0, ties=0, K=0, N=0)
        return out
    if test == "cone":
        K, V, w = cfg["cone"]
        res = enumerate_lifted(K, V, w, rank_begin, rank_end, "cone")
    else:
        pts, w = cfg["affine"]
        K = cfg["dim"] + 1
        res = enumerate_lifted(K, pts, w, rank_begin, rank_end, "affine")
        V = pts
    out.update(degree=res["volume"], cells=res["cells"], singular=res["singular"],
               candidates=res["candidates"], ties=res["ties"], K=K, N=len(V))
    return out
