"""Smith Normal Form by Bezout steps — PAPER.md §3.

Test infrastructure only (see oracle/__init__.py).

P A Q = diag(d_1..d_r, 0..0) with P, Q unimodular (eq. smith).
The reduction follows P:531-568 literally: for a pair of entries a1, a2 with
d = gcd(a1, a2) = s a1 + t a2, the 2x2 unimodular row step
    [[s, t], [-a2/d, a1/d]]
maps (a1, a2)^T to (d, 0)^T, and the column step
    [[s, -a2/d], [t, a1/d]]
maps (a1, a2) to (d, 0).  Repeated row and column steps with
permutations bring A to diagonal form; the divisibility chain
d_1 | ... | d_r is not enforced.  Pivot = entry of minimum
absolute value in the trailing block.

All arithmetic is on Python ints (exact).
"""
from __future__ import annotations

from fractions import Fraction


def ext_gcd(a: int, b: int):
    """Return (g, s, t) with g = gcd(a, b) = s*a + t*b, g > 0 (Bezout).
    When a | b the trivial coefficients (s, t) = (sign a, 0) are returned, so a
    row step with a dividing pivot is a pure elimination."""
    if a != 0 and b % a == 0:
        return abs(a), (1 if a > 0 else -1), 0
    old_r, r = a, b
    old_s, s = 1, 0
    old_t, t = 0, 1
    while r != 0:
        q = old_r // r
        old_r, r = r, old_r - q * r
        old_s, s = s, old_s - q * s
        old_t, t = t, old_t - q * t
    if old_r < 0:
        old_r, old_s, old_t = -old_r, -old_s, -old_t
    return old_r, old_s, old_t


def identity(n: int):
    return [[1 if i == j else 0 for j in range(n)] for i in range(n)]


def _row_step(M, i1, i2, s, t, u, v):
    """rows (i1, i2) <- [[s, t], [u, v]] (rows i1, i2)."""
    r1, r2 = M[i1], M[i2]
    M[i1] = [s * a + t * b for a, b in zip(r1, r2)]
    M[i2] = [u * a + v * b for a, b in zip(r1, r2)]


def _col_step(M, j1, j2, s, t, u, v):
    """cols (j1, j2) <- cols (j1, j2) [[s, u], [t, v]]: new_j1 = s c1 + t c2,
    new_j2 = u c1 + v c2."""
    for row in M:
        a, b = row[j1], row[j2]
        row[j1] = s * a + t * b
        row[j2] = u * a + v * b


def smith_normal_form(A):
    """Return (P, D, Q, r) with P A Q = D diagonal, P and Q unimodular,
    r = rank A.  A: list of n rows of m ints (m may be 0)."""
    n = len(A)
    m = len(A[0]) if n else 0
    M = [list(map(int, row)) for row in A]
    P = identity(n)
    Q = identity(m)
    r = 0
    while r < min(n, m):
        # pivot: minimum |entry| in the trailing block
        best = None
        for i in range(r, n):
            for j in range(r, m):
                if M[i][j] != 0 and (best is None or abs(M[i][j]) < abs(M[best[0]][best[1]])):
                    best = (i, j)
        if best is None:
            break
        bi, bj = best
        if bi != r:
            M[r], M[bi] = M[bi], M[r]
            P[r], P[bi] = P[bi], P[r]
        if bj != r:
            for row in M:
                row[r], row[bj] = row[bj], row[r]
            for row in Q:
                row[r], row[bj] = row[bj], row[r]
        while True:
            # row steps: clear column r below the pivot
            for i in range(r + 1, n):
                if M[i][r] != 0:
                    a1, a2 = M[r][r], M[i][r]
                    g, s, t = ext_gcd(a1, a2)
                    _row_step(M, r, i, s, t, -a2 // g, a1 // g)
                    _row_step(P, r, i, s, t, -a2 // g, a1 // g)
            # column steps: clear row r right of the pivot
            for j in range(r + 1, m):
                if M[r][j] != 0:
                    a1, a2 = M[r][r], M[r][j]
                    g, s, t = ext_gcd(a1, a2)
                    _col_step(M, r, j, s, t, -a2 // g, a1 // g)
                    _col_step(Q, r, j, s, t, -a2 // g, a1 // g)
            if all(M[i][r] == 0 for i in range(r + 1, n)):
                break
        r += 1
    return P, M, Q, r


def matmul(X, Y):
    if not X:
        return []
    inner = len(Y)
    cols = len(Y[0]) if inner else 0
    if inner == 0:
        return [[0] * 0 for _ in X] if not cols else [[0] * cols for _ in X]
    return [[sum(X[i][k] * Y[k][j] for k in range(inner)) for j in range(cols)] for i in range(len(X))]


def det_fraction(M) -> Fraction:
    """Determinant by Gaussian elimination over Q (textbook; Fractions)."""
    n = len(M)
    if n == 0:
        return Fraction(1)
    a = [[Fraction(x) for x in row] for row in M]
    det = Fraction(1)
    for c in range(n):
        p = next((i for i in range(c, n) if a[i][c] != 0), None)
        if p is None:
            return Fraction(0)
        if p != c:
            a[c], a[p] = a[p], a[c]
            det = -det
        det *= a[c][c]
        for i in range(c + 1, n):
            if a[i][c] != 0:
                f = a[i][c] / a[c][c]
                a[i] = [x - f * y for x, y in zip(a[i], a[c])]
    return det


def rank_fraction(M) -> int:
    """Rank over Q by Gaussian elimination (independent of the SNF)."""
    a = [[Fraction(x) for x in row] for row in M]
    n = len(a)
    m = len(a[0]) if n else 0
    r = 0
    for c in range(m):
        p = next((i for i in range(r, n) if a[i][c] != 0), None)
        if p is None:
            continue
        a[r], a[p] = a[p], a[r]
        for i in range(n):
            if i != r and a[i][c] != 0:
                f = a[i][c] / a[r][c]
                a[i] = [x - f * y for x, y in zip(a[i], a[r])]
        r += 1
        if r == n:
            break
    return r
