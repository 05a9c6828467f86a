"""Seeded, synthetic input generators shared by the oracle, the tests and bench.py.

This module holds NONE of the method's arithmetic (no Smith form, no kernel
basis, no determinant, no lifting test).  It only *writes down* binomial
systems x^A = b (eq. standard-form) and point
configurations, and draws the random numbers the method consumes (the
lifting) from a counter-based generator, so that the oracle
(`oracle/`) and the CUDA path (`paper_1501_02237_b200/`) receive bit-identical
inputs without sharing any code.

Conventions:
  * A is returned as a list of n rows, each a list of m Python ints
    (row i = variable x_i, column j = equation j = alpha^(j) - beta^(j)).
  * b is a list of m complex numbers (b_j = -c_{j,2}/c_{j,1}).
  * A lifting is a list of n+1 ints: one per variable, the last one for the
    origin (Prop. 4 includes the origin).
"""
from __future__ import annotations

import math
from itertools import combinations, combinations_with_replacement

MASK64 = (1 << 64) - 1


class SplitMix64:
    """SplitMix64; all arithmetic mod 2^64."""

    def __init__(self, seed: int):
        self.s = seed & MASK64

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform_int(self, lo: int, hi: int) -> int:
        return lo + self.next() % (hi - lo + 1)

    def lift(self) -> int:
        """Uniform integer in [0, 2^20) (SPEC S:298 reading, Z4)."""
        return self.next() >> 44

    def unit_circle(self) -> complex:
        t = (self.next() >> 11) * (2.0 * math.pi / float(1 << 53))
        return complex(math.cos(t), math.sin(t))


def liftings(n_points: int, seed: int) -> list[int]:
    """n_points draws of SplitMix64(seed).lift(), in point order."""
    rng = SplitMix64(seed)
    return [rng.lift() for _ in range(n_points)]


def derive_seed(seed: int, attempt: int) -> int:
    """Seed for re-lift attempt `attempt` (>=1); attempt 0 is `seed` itself.

    Mixing is one SplitMix64 step of (seed ^ attempt*golden); both the oracle
    and the C++ planner implement it (it is input generation, not method)."""
    if attempt == 0:
        return seed & MASK64
    return SplitMix64((seed ^ ((attempt * 0x9E3779B97F4A7C15) & MASK64)) & MASK64).next()


# ---------------------------------------------------------------------------
# Polynomial -> binomial system plumbing (writing down dW = 0)
# ---------------------------------------------------------------------------

def _binomial_system_from_polys(polys, n):
    """polys: list of dict{exponent tuple: coefficient}.  Each non-zero poly
    must have exactly two terms c1 x^alpha + c2 x^beta; it becomes the column
    alpha - beta with b = -c2/c1.  Identically-zero polys are
    skipped (conifold-like cases)."""
    cols, bs = [], []
    for p in polys:
        terms = [(e, c) for e, c in p.items() if c != 0]
        if not terms:
            continue
        if len(terms) != 2:
            raise ValueError("not a binomial: %r" % (terms,))
        (ea, ca), (eb, cb) = sorted(terms)
        cols.append([ea[i] - eb[i] for i in range(n)])
        bs.append(complex(-cb / ca))
    A = [[cols[j][i] for j in range(len(cols))] for i in range(n)]
    return A, bs


def _gradient(terms, n):
    """terms: list of (coeff, exponent tuple).  Returns [dW/dx_v for v]."""
    out = []
    for v in range(n):
        d = {}
        for c, e in terms:
            if e[v] == 0:
                continue
            e2 = list(e)
            e2[v] -= 1
            key = tuple(e2)
            d[key] = d.get(key, 0) + c * e[v]
        out.append(d)
    return out


def master_space_terms(m: int, k: int):
    """Monomials of W_{m,k}, periodic indices i mod m, j mod k
    (reading Z7).  Variable order: x_{i,j}, then y_{i,j}, then
    z_{i,j}, each (i,j) lexicographic."""
    n = 3 * m * k

    def xi(i, j):
        return (i % m) * k + (j % k)

    def yi(i, j):
        return m * k + (i % m) * k + (j % k)

    def zi(i, j):
        return 2 * m * k + (i % m) * k + (j % k)

    terms = []
    for i in range(m):
        for j in range(k):
            e1 = [0] * n
            e1[xi(i, j)] += 1
            e1[yi(i + 1, j)] += 1
            e1[zi(i + 1, j + 1)] += 1
            e2 = [0] * n
            e2[yi(i, j)] += 1
            e2[xi(i, j + 1)] += 1
            e2[zi(i + 1, j + 1)] += 1
            terms.append((1, tuple(e1)))
            terms.append((-1, tuple(e2)))
    return terms, n


def master_space_system(m: int, k: int):
    """grad W_{m,k} = 0 as x^A = b.  Returns (A, b)."""
    terms, n = master_space_terms(m, k)
    return _binomial_system_from_polys(_gradient(terms, n), n)


def dp0_system():
    """C^3/Z_3 (dP0) quiver: W = eps_{ijk} X^i Y^j Z^k, 9 fields (X1..3,
    Y1..3, Z1..3).  SURVEY Z11."""
    n = 9
    terms = []
    for (i, j, kk) in [(0, 1, 2), (1, 2, 0), (2, 0, 1), (0, 2, 1), (2, 1, 0), (1, 0, 2)]:
        sign = 1 if (i, j, kk) in [(0, 1, 2), (1, 2, 0), (2, 0, 1)] else -1
        e = [0] * n
        e[i] += 1
        e[3 + j] += 1
        e[6 + kk] += 1
        terms.append((sign, tuple(e)))
    return _binomial_system_from_polys(_gradient(terms, n), n)


def conifold_system():
    """Conifold W = A1 B1 A2 B2 - A1 B2 A2 B1 (abelian fields commute, so W = 0
    and every F-term vanishes): n = 4, m = 0.  SURVEY Z11."""
    terms = [(1, (1, 1, 1, 1)), (-1, (1, 1, 1, 1))]
    return _binomial_system_from_polys(_gradient(terms, 4), 4)


def _quadric(n, i, j, k, l):
    """Binomial x_i x_j - x_k x_l as a polynomial dict."""
    e1 = [0] * n
    e1[i] += 1
    e1[j] += 1
    e2 = [0] * n
    e2[k] += 1
    e2[l] += 1
    return {tuple(e1): 1, tuple(e2): -1} if tuple(e1) != tuple(e2) else {}


def rnc_system(delta: int):
    """Rational normal curve of degree delta in P^delta: 2x2 minors
    x_i x_{j+1} - x_{i+1} x_j, 0 <= i < j <= delta-1 (degree delta)."""
    n = delta + 1
    polys = [_quadric(n, i, j + 1, i + 1, j) for i in range(delta) for j in range(i + 1, delta)]
    return _binomial_system_from_polys(polys, n)


def twisted_cubic_system():
    """n = 4, A columns (1,-2,1,0), (0,1,-2,1), (1,-1,-1,1), b = 1."""
    cols = [(1, -2, 1, 0), (0, 1, -2, 1), (1, -1, -1, 1)]
    A = [[c[i] for c in cols] for i in range(4)]
    return A, [1 + 0j] * 3


def segre_system(a: int, bdim: int):
    """Segre P^a x P^b: variables x_{ij} (i<=a, j<=b) row-major, binomials
    x_{ij} x_{kl} - x_{il} x_{kj} (degree C(a+b, a))."""
    n = (a + 1) * (bdim + 1)

    def v(i, j):
        return i * (bdim + 1) + j

    polys = []
    for i, kk in combinations(range(a + 1), 2):
        for j, l in combinations(range(bdim + 1), 2):
            polys.append(_quadric(n, v(i, j), v(kk, l), v(i, l), v(kk, j)))
    return _binomial_system_from_polys(polys, n)


def veronese_system(e: int, a: int):
    """Veronese v_e(P^a): variables = degree-e monomials in a+1 variables
    (lexicographic), binomials x_alpha x_beta - x_gamma x_delta for
    alpha+beta = gamma+delta (degree e^a)."""
    monos = sorted(combinations_with_replacement(range(a + 1), e))
    n = len(monos)
    pairs = {}
    for p, q in combinations_with_replacement(range(n), 2):
        key = tuple(sorted(monos[p] + monos[q]))
        pairs.setdefault(key, []).append((p, q))
    polys = []
    for plist in pairs.values():
        for (p, q), (r, s) in combinations(plist, 2):
            polys.append(_quadric(n, p, q, r, s))
    return _binomial_system_from_polys(polys, n)


def c2_system(seed: int):
    """n = 12, m = 8, A uniform in [-3,3] drawn
    column by column; then 13 liftings (12 variables, then the origin); then
    b on the unit circle.  Returns (A, b, lifting)."""
    rng = SplitMix64(seed)
    n, m = 12, 8
    A = [[0] * m for _ in range(n)]
    for j in range(m):
        for i in range(n):
            A[i][j] = rng.uniform_int(-3, 3)
    lifting = [rng.lift() for _ in range(n + 1)]
    b = [rng.unit_circle() for _ in range(m)]
    return A, b, lifting


def c5_points(seed: int, n_points: int = 40, dim: int = 7, lo: int = -3, hi: int = 3):
    """n_points distinct a in [lo,hi]^dim, V_l = (1, a_l)
    in generation order, then n_points liftings.  Returns (V point-major
    list of (dim+1)-tuples, lifting list)."""
    if n_points > (hi - lo + 1) ** dim:
        raise ValueError("not enough distinct lattice points in the box")
    rng = SplitMix64(seed)
    seen, pts = set(), []
    while len(pts) < n_points:
        a = tuple(rng.uniform_int(lo, hi) for _ in range(dim))
        if a not in seen:
            seen.add(a)
            pts.append(a)
    V = [(1,) + a for a in pts]
    lifting = [rng.lift() for _ in range(n_points)]
    return V, lifting


def random_point_set(seed: int, d: int, n_points: int, lo: int = -3, hi: int = 3):
    """Random affine point set in Z^d (possibly with repeats) for route-2
    cross-checks (SPEC S:477 style).  Returns (points, lifting)."""
    rng = SplitMix64(seed)
    pts = [tuple(rng.uniform_int(lo, hi) for _ in range(d)) for _ in range(n_points)]
    lifting = [rng.lift() for _ in range(n_points)]
    return pts, lifting


UNIT_SQUARE = [(0, 0), (0, 1), (1, 1), (1, 0)]  # P:735 example


def named_system(name: str):
    """Registry used by tests / bench: returns (A, b)."""
    if name == "twisted_cubic":
        return twisted_cubic_system()
    if name == "conifold":
        return conifold_system()
    if name == "dp0":
        return dp0_system()
    if name.startswith("W"):
        m, k = name[1:].split("_")
        return master_space_system(int(m), int(k))
    if name.startswith("rnc"):
        return rnc_system(int(name[3:]))
    raise KeyError(name)
