"""Structure of V*(x^A - b) from the Smith form — PAPER.md §2.

Test infrastructure only (see oracle/__init__.py).

Prop. 1: #components = |prod d_j|, codim = r = rank A.
eq. rank-decomp: P = [P_r; P_0] (top r rows / last n-r rows),
Q = [Q_r, Q_0] (left r columns / remaining m-r columns).
eq. consistency: if r < m the system is consistent iff
b^{Q_0} = 1; checked to 1e-8 for complex b (SPEC S:163 reading).
P:384-388: r = n gives isolated points (dimension 0).
"""
from __future__ import annotations

import cmath

from .snf import smith_normal_form

CONSISTENCY_TOL = 1e-8


def b_power(b, Q0col):
    """prod_i b_i^{Q0[i]} for integer exponents (eq. matrix-power)."""
    out = complex(1.0)
    for bi, e in zip(b, Q0col):
        if e:
            out *= complex(bi) ** e
    return out


def analyze(A, b=None):
    """Return dict(n, m, rank, dim, components, P0, consistent, D) (Props 1-2)."""
    n = len(A)
    m = len(A[0]) if n else 0
    P, D, Q, r = smith_normal_form(A)
    comps = 1
    for j in range(r):
        comps *= D[j][j]
    comps = abs(comps)
    P0 = [row[:] for row in P[r:]]                    # last n-r rows
    Q0 = [[Q[i][j] for j in range(r, m)] for i in range(m)]  # last m-r cols
    consistent = True
    if r < m:
        bb = b if b is not None else [1.0] * m
        for k in range(m - r):
            val = b_power(bb, [Q0[i][k] for i in range(m)])
            if abs(val - 1.0) > CONSISTENCY_TOL * max(1.0, abs(val)):
                consistent = False
    return {
        "n": n, "m": m, "rank": r, "dim": n - r, "components": comps,
        "P": P, "Q": Q, "D": [D[j][j] for j in range(r)], "P0": P0,
        "consistent": consistent,
    }


__all__ = ["analyze", "b_power", "cmath"]
