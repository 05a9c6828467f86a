"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Nothing here touches the CUDA path.  Each test names the passage or the
mathematical fact it checks; a plausible mistake in the oracle (dropped
origin, wrong sign in the lower-face test, transposed P0, wrong rank order)
fails at least one of them.
"""
import itertools
import math
from fractions import Fraction

import pytest

import workloads as W
from oracle import (analyze, colex_rank, colex_unrank, degree, det_fraction,
                    enumerate_lifted, nvol_pulling, rank_fraction,
                    smith_normal_form)
from oracle.native import enumerate_range
from oracle.points import point_configuration
from oracle.snf import ext_gcd, matmul
from oracle.subdivision import colex_next, lower_face_affine

from conftest import golden


# ----------------------------------------------------------------- SNF (§3)

def _gcd_of_minors(A, r):
    n, m = len(A), len(A[0])
    g = 0
    for rows in itertools.combinations(range(n), r):
        for cols in itertools.combinations(range(m), r):
            g = math.gcd(g, int(det_fraction([[A[i][j] for j in cols] for i in rows])))
    return g


def test_bezout_step_example():
    # P = [[s, t], [-a2/d, a1/d]] maps (a1, a2)^T to (d, 0)^T, det P = 1
    for a1, a2 in [(4, 6), (6, 4), (-9, 12), (5, 7), (3, 9), (0, 5)]:
        if a1 == 0:
            continue
        g, s, t = ext_gcd(a1, a2)
        P = [[s, t], [-a2 // g, a1 // g]]
        assert matmul(P, [[a1], [a2]]) == [[g], [0]]
        assert s * (a1 // g) + t * (a2 // g) == 1
        assert g == math.gcd(a1, a2)


def test_snf_properties_random():
    # eq. smith: P A Q diagonal, P, Q unimodular; rank = rank over Q;
    # prod d_j = gcd of the r x r minors (the r-th determinantal divisor)
    rng = W.SplitMix64(7)
    for trial in range(60):
        n = 1 + rng.uniform_int(0, 4)
        m = 1 + rng.uniform_int(0, 4)
        A = [[rng.uniform_int(-4, 4) for _ in range(m)] for _ in range(n)]
        if trial % 7 == 0:  # force rank deficiency
            A[-1] = [2 * x for x in A[0]]
        P, D, Q, r = smith_normal_form(A)
        PAQ = matmul(matmul(P, A), Q)
        assert PAQ == D
        for i in range(n):
            for j in range(m):
                if i != j or i >= r:
                    assert D[i][j] == 0
                else:
                    assert D[i][j] != 0
        assert abs(det_fraction(P)) == 1 and abs(det_fraction(Q)) == 1
        assert r == rank_fraction(A)
        if r > 0:
            prod = abs(math.prod(D[j][j] for j in range(r)))
            assert prod == _gcd_of_minors(A, r)


def test_components_diag():
    # SPEC S:126 / Prop. 1: A = diag(2,3) -> 6 isolated points
    info = analyze([[2, 0], [0, 3]])
    assert info["rank"] == 2 and info["dim"] == 0 and info["components"] == 6
    r = degree([[2, 0], [0, 3]])
    assert r["degree"] == 1  # dimension 0 -> points (degree 1 each)


def test_identity_system_dim0():
    r = degree([[1, 0], [0, 1]], [1, 1])
    assert r["dim"] == 0 and r["components"] == 1 and r["degree"] == 1


def test_inconsistent_system():
    # eq. consistency: x1 = 1 and x1 = 2 is inconsistent
    A = [[1, 1], [0, 0]]
    assert not analyze(A, [1, 2])["consistent"]
    assert analyze(A, [2, 2])["consistent"]
    assert degree(A, [1, 2])["degree"] is None


def test_p0_is_left_kernel_basis():
    # eq. rank-decomp: P0 A = 0 and P0 has full row rank d
    for m, k in [(1, 2), (2, 2), (2, 3)]:
        A, b = W.master_space_system(m, k)
        info = analyze(A, b)
        P0 = info["P0"]
        assert matmul(P0, A) == [[0] * len(A[0]) for _ in P0]
        assert rank_fraction(P0) == info["dim"]


def test_table1_dimensions():
    # Table 1, P:1602-1621 (tests/golden/table1_dims.txt)
    rows = {}
    with open(golden("table1_dims.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            m, vals = line.split(":")
            rows[int(m)] = [int(v) for v in vals.split()]
    for m, vals in rows.items():
        for k, want in enumerate(vals, start=1):
            if want < 0:
                continue
            A, b = W.master_space_system(m, k)
            info = analyze(A, b)
            assert info["dim"] == want, (m, k)
            assert info["components"] == 1          # conjecture


def test_table2_dimensions_small():
    # Table 2, the entries the Python SNF finishes in seconds
    with open(golden("table2_dims.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            m, want = map(int, line.split())
            if m > 10:
                continue
            A, b = W.master_space_system(m, m)
            assert analyze(A, b)["dim"] == want


# ----------------------------------------------------- rank order (§8.a3)

def test_colex_rank_roundtrip():
    for N, K in [(6, 3), (9, 4), (12, 1), (7, 7)]:
        combos = sorted(itertools.combinations(range(N), K), key=lambda c: tuple(reversed(c)))
        for r, c in enumerate(combos):
            assert colex_rank(c) == r
            assert colex_unrank(r, K) == c
        c = combos[0]
        for r in range(1, len(combos)):
            c = colex_next(c, N)
            assert c == combos[r]
        assert colex_next(c, N) is None


# --------------------------------------------- degree = volume (§4, Prop 4)

def _closed_form_system(name):
    if name.startswith("segre"):
        a, b2 = name[5:].split("x")
        return W.segre_system(int(a), int(b2))
    if name.startswith("veronese"):
        e, a = name[8:].split("_")
        return W.veronese_system(int(e), int(a))
    return W.named_system(name)


def test_closed_forms():
    with open(golden("closed_forms.txt")) as f:
        items = [l.split() for l in f if l.strip() and not l.startswith("#")]
    for name, want in items:
        want = int(want)
        if name == "unit_square":
            assert nvol_pulling(W.UNIT_SQUARE) == want
            continue
        A, b = _closed_form_system(name)
        n = len(A)
        r = degree(A, b, W.liftings(n + 1, 3))
        assert r["ties"] == 0
        assert r["degree"] == want, name
        assert r["components"] == 1


def test_unit_square_worked_example():
    # S = {(0,0),(0,1),(1,1),(1,0)} lifted generically -> two triangles
    pts = W.UNIT_SQUARE
    # liftings (1,0,1,0): (0,0) and (1,1) lifted above the plane of the others
    cells = [c for c in itertools.combinations(range(4), 3)
             if lower_face_affine(pts, [1, 0, 1, 0], c)[0] == "cell"]
    assert sorted(cells) == [(0, 1, 3), (1, 2, 3)]
    assert sum(lower_face_affine(pts, [1, 0, 1, 0], c)[1] for c in cells) == 2
    # SPEC's (1,0,0,1) lifting is degenerate: all four lifted points coplanar
    st = [lower_face_affine(pts, [1, 0, 0, 1], c)[0] for c in itertools.combinations(range(4), 3)]
    assert "cell" not in st and "tie" in st
    # cone formulation of the same (V = (1, a)) agrees
    V = [(1,) + p for p in pts]
    res = enumerate_lifted(3, V, [1, 0, 1, 0])
    assert res["volume"] == 2 and res["cells"] == 2 and res["ties"] == 0


def test_table3_small_python(table3):
    # Table 3: entries the Fraction oracle finishes quickly
    for (m, k) in [(1, 2), (1, 3), (1, 4), (2, 1), (3, 1), (2, 2)]:
        A, b = W.master_space_system(m, k)
        r = degree(A, b, W.liftings(len(A) + 1, 1))
        assert r["degree"] == table3[(m, k)][0], (m, k)
        assert r["ties"] == 0


def test_table3_c_oracle(table3):
    # Table 3 entries via the C variant of the same brute force
    for (m, k) in [(1, 5), (1, 6), (1, 7), (4, 1), (5, 1), (2, 3), (3, 2), (2, 4)]:
        A, b = W.master_space_system(m, k)
        cfg = point_configuration(A, b, W.liftings(len(A) + 1, 1))
        K, V, w = cfg["cone"]
        r = enumerate_range(K, V, w, threads=8)
        assert r["status"] == 0 and r["ties"] == 0
        assert r["volume"] == table3[(m, k)][0], (m, k)


def test_conjecture_recurrence_w2k():
    # Conjecture: deg W_{2,k} = 6 deg W_{2,k-1} + 2^{2k-3}
    vals = {}
    for k in (2, 3, 4):
        A, b = W.master_space_system(2, k)
        cfg = point_configuration(A, b, W.liftings(len(A) + 1, 2))
        K, V, w = cfg["cone"]
        vals[k] = enumerate_range(K, V, w, threads=8)["volume"]
    assert vals[3] == 6 * vals[2] + 2 ** 3
    assert vals[4] == 6 * vals[3] + 2 ** 5


# ----------------------------------------------------- invariances

def test_lifting_invariance_and_cells_bound():
    # the subdivision depends on the lifting, its volume does not;
    # every cell has NVol >= 1 so cells <= degree
    A, b = W.master_space_system(2, 3)
    degs = set()
    for seed in (1, 2, 3, 4):
        cfg = point_configuration(A, b, W.liftings(len(A) + 1, seed))
        K, V, w = cfg["cone"]
        r = enumerate_range(K, V, w, threads=4)
        degs.add(r["volume"])
        assert r["cells"] <= r["volume"]
    assert degs == {92}


def test_singular_count_lifting_independent():
    # det V_sigma does not involve the lifting
    A, b = W.master_space_system(2, 2)
    sing = set()
    for seed in (1, 5, 9):
        r = degree(A, b, W.liftings(len(A) + 1, seed))
        sing.add(r["singular"])
    assert len(sing) == 1


def test_homogeneous_shortcut_matches_generic():
    # points.py reading: K = d (pyramid) and K = d+1 with the origin agree
    for name in ["twisted_cubic", "dp0", "W1_3", "W2_2", "rnc4"]:
        A, b = W.named_system(name)
        lift = W.liftings(len(A) + 1, 5)
        r1 = degree(A, b, lift, test="cone")
        r2 = degree(A, b, lift, test="affine")
        assert r1["homogeneous"]
        assert r1["K"] == r1["dim"] and r2["K"] == r1["dim"] + 1
        assert r1["degree"] == r2["degree"]


def test_variable_and_equation_permutation():
    A, b = W.master_space_system(2, 2)
    n, m = len(A), len(A[0])
    rng = W.SplitMix64(11)
    perm_r = list(range(n))
    perm_c = list(range(m))
    for i in range(n - 1, 0, -1):
        j = rng.uniform_int(0, i)
        perm_r[i], perm_r[j] = perm_r[j], perm_r[i]
    for i in range(m - 1, 0, -1):
        j = rng.uniform_int(0, i)
        perm_c[i], perm_c[j] = perm_c[j], perm_c[i]
    A2 = [[A[perm_r[i]][perm_c[j]] for j in range(m)] for i in range(n)]
    r1 = degree(A, b, W.liftings(n + 1, 1))
    r2 = degree(A2, [b[j] for j in perm_c], W.liftings(n + 1, 1))
    assert r1["degree"] == r2["degree"] == 14


def test_unimodular_change_of_points():
    # NVol is GL_d(Z)-invariant, and so is the whole lifted test (cells identical)
    rng = W.SplitMix64(3)
    for trial in range(10):
        pts, w = W.random_point_set(100 + trial, 3, 8)
        pts = list(dict.fromkeys(pts))
        w = w[:len(pts)]
        if rank_fraction([[p[t] - pts[0][t] for t in range(3)] for p in pts]) < 3:
            continue
        G = [[1, 0, 0], [0, 1, 0], [0, 0, 1]]
        for _ in range(6):  # random elementary unimodular operations
            i, j = rng.uniform_int(0, 2), rng.uniform_int(0, 2)
            if i != j:
                c = rng.uniform_int(-2, 2)
                G[i] = [x + c * y for x, y in zip(G[i], G[j])]
        pts2 = [tuple(sum(G[i][t] * p[t] for t in range(3)) for i in range(3)) for p in pts]
        V1 = [(1,) + p for p in pts]
        V2 = [(1,) + p for p in pts2]
        assert enumerate_lifted(4, V1, w) == enumerate_lifted(4, V2, w)


def test_route1_vs_route2_random_sets():
    # SPEC S:477 / SURVEY §8.c route 2: the lifted brute force equals an
    # independent pulling-triangulation volume (no lifting at all)
    checked = 0
    for seed in range(400):
        d = 1 + seed % 4
        n_pts = d + 2 + (seed % 5)
        pts, w = W.random_point_set(seed, d, n_pts, -2, 2)
        pts = list(dict.fromkeys(pts))
        if len(pts) <= d:
            continue
        if rank_fraction([[p[t] - pts[0][t] for t in range(d)] for p in pts]) < d:
            continue
        w = W.liftings(len(pts), 1000 + seed)
        V = [(1,) + p for p in pts]
        r = enumerate_lifted(d + 1, V, w)
        assert r["ties"] == 0
        assert r["volume"] == nvol_pulling(pts), (seed, pts)
        checked += 1
        if checked >= 60:
            break
    assert checked >= 60


def test_degenerate_lifting_detected():
    # constant lifting: every lifted point is on one hyperplane, so any
    # configuration with more than K points has ties (reading Z3)
    V, _ = W.c5_points(4, n_points=10, dim=3)
    r = enumerate_lifted(4, V, [7] * 10)
    assert r["ties"] > 0


def test_c_oracle_matches_python_oracle():
    cases = []
    for name in ["twisted_cubic", "dp0", "W1_3", "W2_2", "rnc6"]:
        A, b = W.named_system(name)
        cfg = point_configuration(A, b, W.liftings(len(A) + 1, 1))
        cases.append(cfg["cone"])
    for s in (5, 31):
        A, b, lift = W.c2_system(s)
        cases.append(point_configuration(A, b, lift)["cone"])
    V, w = W.c5_points(1, n_points=14, dim=4)
    cases.append((5, V, w))
    V, w = W.c5_points(9, n_points=10, dim=3)
    cases.append((4, V, [3] * 10))                       # degenerate lifting
    for K, V, w in cases:
        py = enumerate_lifted(K, V, w)
        c = enumerate_range(K, V, w, threads=2)
        assert c["status"] == 0
        for key in py:
            assert py[key] == c[key], (K, key)
        total = math.comb(len(V), K)
        for (b, e) in [(0, total // 3), (total // 3, total - 1), (total // 2, total // 2 + 7)]:
            py = enumerate_lifted(K, V, w, b, e)
            c = enumerate_range(K, V, w, b, e, threads=3)
            assert all(py[k] == c[k] for k in py)
    # the C variant itself (no Python fallback) on cases that fit __int128
    assert all(enumerate_range(K, V, w).get("fallback", 0) == 0 for K, V, w in cases[:5])


def test_c2_components_and_invariance():
    # C2: seeds 5/31/46/66 have rank 8 and prod d_j > 1;
    # degree invariant under the lifting; route 1 (cone) == route 1 (affine)
    for s in (5, 31):
        A, b, lift = W.c2_system(s)
        info = analyze(A, b)
        assert info["rank"] == 8 and info["components"] > 1
        r1 = degree(A, b, lift)
        r2 = degree(A, b, W.liftings(13, 77))
        assert r1["degree"] == r2["degree"] and r1["ties"] == 0


def test_cell_list_is_a_subdivision():
    # Def. 1: the cells cover conv S with disjoint interiors, so
    # their volumes add up to NVol (route 2) and every cell is affinely
    # independent (NVol >= 1)
    from oracle import cell_list
    for seed in range(8):
        pts, _ = W.random_point_set(300 + seed, 2 + seed % 2, 9, -2, 2)
        pts = list(dict.fromkeys(pts))
        d = len(pts[0])
        if rank_fraction([[p[t] - pts[0][t] for t in range(d)] for p in pts]) < d:
            continue
        V = [(1,) + p for p in pts]
        w = W.liftings(len(V), 900 + seed)
        cells = cell_list(d + 1, V, w)
        assert all(v >= 1 for _, v in cells)
        assert sum(v for _, v in cells) == nvol_pulling(pts)
        assert len(cells) == enumerate_lifted(d + 1, V, w)["cells"]


def _delaunay_case(seed, d, n, lo, hi):
    """Distinct random integer points with the paraboloid lifting |p|^2: the
    lower faces of the lifted set project to the Delaunay triangulation
    (the regular subdivision of Def. 1, for this lifting)."""
    pts, _ = W.random_point_set(seed, d, n, lo, hi)
    pts = list(dict.fromkeys(pts))
    w = [sum(x * x for x in p) for p in pts]
    return pts, [(1,) + p for p in pts], w


def _on_hull_boundary(pts):
    # brute force in the plane: p is on the boundary of conv(pts) iff some
    # line through p and another point q leaves every point on one side
    out = 0
    for i, p in enumerate(pts):
        for j, q in enumerate(pts):
            if i == j:
                continue
            s = [(q[0] - p[0]) * (r[1] - p[1]) - (q[1] - p[1]) * (r[0] - p[0]) for r in pts]
            if all(x >= 0 for x in s) or all(x <= 0 for x in s):
                out += 1
                break
    return out


def test_cells_are_delaunay_for_paraboloid_lifting():
    # Independent pin of the oracle's cell LIST (not only its volume sum):
    # with the lifting w(p) = |p|^2 the regular subdivision is the Delaunay
    # triangulation, computed here by qhull (scipy), which shares nothing with
    # the lower-face test of P:782-792.  In the plane every point is a vertex,
    # so Euler's formula fixes the count: #triangles = 2n - b - 2 (b = points
    # on the hull boundary).  Seeds with cospherical points (ties) are skipped.
    spatial = pytest.importorskip("scipy.spatial")
    from oracle import cell_list
    checked = {2: 0, 3: 0}
    for seed in range(200):
        d = 2 + seed % 2
        n = (12 + seed % 7) if d == 2 else (9 + seed % 5)
        pts, V, w = _delaunay_case(7000 + seed, d, n, -6 if d == 2 else -4, 6 if d == 2 else 4)
        if rank_fraction([[p[t] - pts[0][t] for t in range(d)] for p in pts]) < d:
            continue
        if enumerate_lifted(d + 1, V, w)["ties"]:
            continue
        tri = spatial.Delaunay(pts)
        if len(tri.coplanar):
            continue
        want = sorted(tuple(sorted(int(i) for i in s)) for s in tri.simplices)
        got = cell_list(d + 1, V, w)
        assert [c for c, _ in got] == want, (seed, pts)
        for c, v in got:                     # NVol = d! * Euclidean volume
            assert v == abs(round(det_fraction([list(V[i]) for i in c])))
        if d == 2:
            assert len(got) == 2 * len(pts) - _on_hull_boundary(pts) - 2
        assert sum(v for _, v in got) == nvol_pulling(pts)
        checked[d] += 1
        if min(checked.values()) >= 15:
            break
    assert checked[2] >= 15 and checked[3] >= 15, checked
