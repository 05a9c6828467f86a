"""The point configuration whose normalised volume is the degree — PAPER.md
Prop. 4 (eq. deg-vol) and §4.

Test infrastructure only (see oracle/__init__.py).

deg V = d! Vol_d(conv{p_0^(1), ..., p_0^(n), 0})

where p_0^(j) are the columns of P_0.  Readings:
  Z2  the origin IS included (Prop. 4 is the theorem; eq. deg-vol2 at P:638
      omits it, which is wrong for e.g. the twisted cubic).
  Z5  S is a set: duplicate columns merge, keeping the minimum
      lifting value.  A zero column coincides with the
      origin and is merged into it.
  Ordering: distinct non-zero columns in order of first occurrence
      (variable order), then the origin last.  The lifting is given per
      variable plus one value for the origin (n+1 values).

Two equivalent descriptions are returned:
  * `affine`: the points a in Z^d of S u {0} with lifts — the paper's own
    objects, used by the paper-literal lower-face test.
  * `cone`: K-vectors V with lifts, the configuration the B200 kernel
    enumerates K-subsets of.  Generic case: V = (1, a), K = d+1 (the
    standard homogenisation: det[(1,a_0)..(1,a_d)] = det(a_1-a_0..a_d-a_0)).
    Homogeneous case (every column of A sums to zero, 1^T A = 0): then
    1^T lies in the row space of P_0 over Q and, the kernel lattice being
    saturated, 1^T = lambda^T P_0 with lambda integral, so every point lies on
    the hyperplane lambda.p = 1.  conv(S u {0}) is then a pyramid with apex 0
    and every full-dimensional simplex of S u {0} contains the apex, so the
    cells are {0} u sigma, |sigma| = d, with NVol = |det[p_sigma]|; V = S,
    K = d (reading "homogeneous shortcut").
"""
from __future__ import annotations

from .binomial import analyze


def point_configuration(A, b=None, lifting=None):
    """Return dict with keys dim, components, consistent, homogeneous,
    affine (points, lifts), cone (K, V point-major, lifts).

    lifting: n+1 ints (variables, then origin) or None (all zero — only
    meaningful for tests of the front end)."""
    info = analyze(A, b)
    n = info["n"]
    d = info["dim"]
    if lifting is None:
        lifting = [0] * (n + 1)
    if len(lifting) != n + 1:
        raise ValueError("lifting must have n+1 entries")
    out = dict(info)
    m = info["m"]
    homog = all(sum(A[i][j] for i in range(n)) == 0 for j in range(m))
    out["homogeneous"] = homog
    if not info["consistent"] or d == 0:
        out["affine"] = None
        out["cone"] = None
        return out
    P0 = info["P0"]
    cols = [tuple(P0[i][j] for i in range(d)) for j in range(n)]
    zero = tuple([0] * d)
    order, lift_of = [], {}
    origin_lift = lifting[n]
    for j, c in enumerate(cols):
        if c == zero:
            origin_lift = min(origin_lift, lifting[j])
            continue
        if c not in lift_of:
            order.append(c)
            lift_of[c] = lifting[j]
        else:
            lift_of[c] = min(lift_of[c], lifting[j])
    pts = list(order) + [zero]
    lifts = [lift_of[c] for c in order] + [origin_lift]
    out["affine"] = (pts, lifts)
    if homog:
        out["cone"] = (d, [tuple(c) for c in order], [lift_of[c] for c in order])
    else:
        out["cone"] = (d + 1, [(1,) + c for c in pts], list(lifts))
    return out
