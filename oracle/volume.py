"""Independent normalised volume, no lifting — the second route for the
oracle (SURVEY §8.c route 2; "facet enumeration + fan
triangulation from a hull vertex").

Test infrastructure only (see oracle/__init__.py).

NVol_d(conv P) for a full-dimensional lattice point set P in Z^d,
computed by a pulling triangulation: pick v = the lexicographically smallest
point (a vertex), triangulate every facet F of conv P not containing v
recursively (inside its own affine hull, again pulling its lexicographically
smallest point), and cone each simplex of F from v.  The d-simplices so
obtained triangulate conv P (standard; de Loera-Rambau-Santos, cited by the
paper at P:669), and NVol = sum |det(s_1 - s_0, ..., s_d - s_0)| (Z1).

Facets are found by brute force: every affinely independent k-subset of the
points of a k-dimensional configuration spans a hyperplane of its affine
hull; it supports a facet iff all points lie weakly on one side.  Only for
tiny inputs (N <= ~14, d <= ~5).  Exact Fractions throughout.
"""
from __future__ import annotations

from fractions import Fraction
from itertools import combinations

from .snf import det_fraction, rank_fraction


def _affine_coords(idx, pts):
    """Coordinates of pts[idx] in a basis of their affine hull.
    Returns (k, {i: tuple of k Fractions})."""
    base = pts[idx[0]]
    diffs = [[Fraction(p - q) for p, q in zip(pts[i], base)] for i in idx]
    # pick a maximal independent subset of the difference vectors
    basis = []
    for i, dv in zip(idx, diffs):
        if rank_fraction(basis + [dv]) > len(basis):
            basis.append(dv)
    k = len(basis)
    coords = {}
    if k == 0:
        return 0, {i: () for i in idx}
    # solve dv = sum lambda_t basis_t via least-squares-free exact elimination:
    # use k coordinates where the basis matrix has full rank
    dim = len(base)
    rows = None
    for cand in combinations(range(dim), k):
        sub = [[basis[t][c] for t in range(k)] for c in cand]
        if det_fraction(sub) != 0:
            rows = cand
            break
    for i, dv in zip(idx, diffs):
        # solve sub * lam = dv[rows]
        sub = [[basis[t][c] for t in range(k)] + [dv[c]] for c in rows]
        lam = _gauss_solve(sub, k)
        coords[i] = tuple(lam)
    return k, coords


def _gauss_solve(aug, k):
    a = [row[:] for row in aug]
    for c in range(k):
        p = next(i for i in range(c, k) if a[i][c] != 0)
        a[c], a[p] = a[p], a[c]
        for i in range(k):
            if i != c and a[i][c] != 0:
                f = a[i][c] / a[c][c]
                a[i] = [x - f * y for x, y in zip(a[i], a[c])]
    return [a[i][k] / a[i][i] for i in range(k)]


def _facets(idx, coords, k):
    """Facets of conv(idx) inside its k-dim affine hull, as frozensets."""
    found = set()
    for sub in combinations(idx, k):
        q0 = coords[sub[0]]
        dirs = [[a - b for a, b in zip(coords[s], q0)] for s in sub[1:]]
        if k > 1 and rank_fraction(dirs) < k - 1:
            continue
        # normal n: n . dir = 0 for all dirs  (k-1 equations, k unknowns),
        # via cofactors of the (k-1) x k matrix
        normal = []
        for t in range(k):
            minor = [[row[u] for u in range(k) if u != t] for row in dirs]
            normal.append(((-1) ** t) * det_fraction(minor))
        sides = []
        on = []
        for i in idx:
            val = sum(nn * (a - b) for nn, a, b in zip(normal, coords[i], q0))
            if val == 0:
                on.append(i)
            else:
                sides.append(val > 0)
        if sides and (all(sides) or not any(sides)):
            found.add(frozenset(on))
        elif not sides:
            raise ValueError("degenerate configuration in facet search")
    return found


def _pull(idx, pts):
    """Pulling triangulation of conv(pts[idx]); returns list of vertex tuples
    (each of size k+1 where k = affine dimension)."""
    idx = sorted(set(idx), key=lambda i: pts[i])
    # drop duplicate points (same coordinates)
    uniq, seen = [], set()
    for i in idx:
        if pts[i] not in seen:
            seen.add(pts[i])
            uniq.append(i)
    idx = uniq
    k, coords = _affine_coords(idx, pts)
    if k == 0:
        return [(idx[0],)]
    v = idx[0]                               # lexicographically smallest point
    if k == 1:
        # segment: endpoints are the extreme coordinates
        lo = min(idx, key=lambda i: coords[i][0])
        hi = max(idx, key=lambda i: coords[i][0])
        return [(lo, hi)]
    out = []
    for F in _facets(idx, coords, k):
        if v in F:
            continue
        for tau in _pull(list(F), pts):
            out.append((v,) + tau)
    return out


def nvol_pulling(points):
    """NVol_d(conv(points)) for points in Z^d (0 if not full-dimensional)."""
    pts = [tuple(int(x) for x in p) for p in points]
    d = len(pts[0])
    idx = list(range(len(pts)))
    k, _ = _affine_coords(idx, pts)
    if k < d:
        return 0
    total = 0
    for s in _pull(idx, pts):
        M = [[pts[s[j]][t] - pts[s[0]][t] for t in range(d)] for j in range(1, d + 1)]
        total += abs(det_fraction(M))
    assert total.denominator == 1
    return int(total)
