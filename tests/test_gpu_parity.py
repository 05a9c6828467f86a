"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element (degree, cells, singular, candidates, ties) on the same
seeded inputs.  All of this is integer work, so the bar is bit-exact.
"""
import math
import random

import pytest

import workloads as W
from oracle import enumerate_lifted, point_configuration
from oracle.native import enumerate_range

B = pytest.importorskip("paper_1501_02237_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

KEYS = ("volume", "cells", "singular", "candidates", "ties")


def _gpu(r):
    return {"volume": r.degree, "cells": r.cells, "singular": r.singular,
            "candidates": r.candidates, "ties": r.ties}


def _oracle_system(A, b, lift, threads=8):
    cfg = point_configuration(A, b, lift)
    K, V, w = cfg["cone"]
    return enumerate_range(K, V, w, threads=threads), cfg


def _assert_same(g, o, what=""):
    for k in KEYS:
        assert g[k] == o[k], (what, k, g, o)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


SYSTEMS = ["twisted_cubic", "conifold", "dp0", "W1_2", "W1_3", "W1_4", "W1_5", "W1_6",
           "W2_1", "W3_1", "W2_2", "W2_3", "rnc3", "rnc7", "rnc20"]


@pytest.mark.parametrize("name", SYSTEMS)
def test_systems_full(name):
    A, b = W.named_system(name)
    lift = W.liftings(len(A) + 1, 1)
    o, cfg = _oracle_system(A, b, lift)
    r = B.Plan.from_system(A, b, lift).degree()
    assert r.K == cfg["cone"][0] and r.N == len(cfg["cone"][1])
    assert r.dim == cfg["dim"] and r.components == cfg["components"]
    _assert_same(_gpu(r), o, name)


@pytest.mark.parametrize("seed", [5, 31, 46, 66])
@pytest.mark.parametrize("flags", [0, 0x1])          # LLL basis and raw SNF basis
def test_c2_random_systems(seed, flags):
    A, b, lift = W.c2_system(seed)
    o, cfg = _oracle_system(A, b, lift)
    r = B.Plan.from_system(A, b, lift, flags=flags).degree()
    assert r.components == cfg["components"] > 1
    _assert_same(_gpu(r), o, seed)


def test_toric_closed_forms():
    for sysf, want in [(W.segre_system(2, 3), 10), (W.veronese_system(2, 3), 8),
                       (W.veronese_system(3, 2), 9), (W.segre_system(1, 4), 5)]:
        A, b = sysf
        lift = W.liftings(len(A) + 1, 2)
        o, _ = _oracle_system(A, b, lift)
        r = B.Plan.from_system(A, b, lift).degree()
        _assert_same(_gpu(r), o)
        assert r.degree == want


@pytest.mark.parametrize("inner", [0, 1, 2, 3])
@pytest.mark.parametrize("tierflag", [0x4, 0x8, 0x20])
def test_inner_levels_and_tiers(inner, tierflag):
    # every register-DFS depth and both arithmetic tiers give identical counts
    for (n_pts, dim, seed) in [(14, 4, 1), (33, 3, 2), (40, 4, 3), (64, 3, 4)]:
        V, w = W.c5_points(seed, n_points=n_pts, dim=dim)
        K = dim + 1
        o = enumerate_range(K, V, w, threads=8)
        r = B.Plan.from_points(V, w, inner_levels=inner, flags=tierflag).degree()
        _assert_same(_gpu(r), o, (n_pts, dim, inner, tierflag))


def test_tier0_overflow_rerun():
    # raw SNF basis of C2 needs > 31-bit values: the int32 tier must hand the
    # affected blocks to tier 2 and still be exact
    A, b, lift = W.c2_system(5)
    o, _ = _oracle_system(A, b, lift)
    r = B.Plan.from_system(A, b, lift, flags=0x1 | 0x4, inner_levels=0).degree()
    assert r.overflow_reruns > 0
    _assert_same(_gpu(r), o)


def test_random_point_sets():
    # SPEC S:477 style: many small random configurations, d <= 4
    rng = random.Random(5)
    done = 0
    for seed in range(300):
        d = 1 + seed % 4
        pts, _ = W.random_point_set(seed, d, d + 2 + seed % 9, -2, 2)
        pts = list(dict.fromkeys(pts))
        if len(pts) < d + 1:
            continue
        V = [(1,) + p for p in pts]
        w = W.liftings(len(V), 500 + seed)
        o = enumerate_lifted(d + 1, V, w)
        if o["volume"] == 0:
            continue
        r = B.Plan.from_points(V, w, inner_levels=rng.randint(0, 3)).degree_range(0, math.comb(len(V), d + 1))
        _assert_same(_gpu(r), o, seed)
        done += 1
    assert done > 100


def test_rank_ranges_c5_full_size():
    # C5: K = 8 over 40 points, 7.7e7 candidates; sampled rank
    # intervals against the oracle, in the launch configuration bench.py uses
    V, w = W.c5_points(1)
    plan = B.Plan.from_points(V, w)
    total = math.comb(40, 8)
    rng = random.Random(11)
    for _ in range(12):
        b = rng.randrange(0, total - 30000)
        e = b + rng.randrange(1, 30000)
        o = enumerate_range(8, V, w, b, e, threads=8)
        r = plan.degree_range(b, e)
        _assert_same(_gpu(r), o, (b, e))
    # the first and last ranks and a tiny interval
    for (b, e) in [(0, 5000), (total - 4000, total), (123456, 123457)]:
        _assert_same(_gpu(plan.degree_range(b, e)), enumerate_range(8, V, w, b, e, threads=8), (b, e))


@pytest.mark.parametrize("mk", [(2, 4), (3, 3), (2, 5)])
def test_master_space_ranges(mk):
    A, b = W.master_space_system(*mk)
    lift = W.liftings(len(A) + 1, 1)
    cfg = point_configuration(A, b, lift)
    # ranks refer to the plan's point order: first occurrence (the oracle's own
    # configuration, FLAG_NATURAL_ORDER) and the default order sorted by lifting
    # residual (the configuration the plan reports, bdeg_plan_points_get)
    plan_nat = B.Plan.from_system(A, b, lift, flags=B.bdeg.FLAG_NATURAL_ORDER)
    plan = B.Plan.from_system(A, b, lift)
    K, V, w = cfg["cone"]
    Kp, Vp, wp = plan.points()
    assert sorted(wp) == sorted(w)                     # the same points, the plan's order
    total = math.comb(len(V), K)
    rng = random.Random(mk[0] * 10 + mk[1])
    for _ in range(6):
        b0 = rng.randrange(0, total - 20000)
        e0 = b0 + rng.randrange(1, 20000)
        _assert_same(_gpu(plan_nat.degree_range(b0, e0)), enumerate_range(K, V, w, b0, e0, threads=8), (b0, e0))
        _assert_same(_gpu(plan.degree_range(b0, e0)), enumerate_range(Kp, Vp, wp, b0, e0, threads=8), (b0, e0))


def test_table3_degrees_gpu(table3):
    # Table 3 exact entries within brute-force reach on one B200
    for mk in [(1, 7), (1, 8), (2, 4), (3, 3), (2, 5), (5, 1), (8, 1)]:
        A, b = W.master_space_system(*mk)
        r = B.degree(A, b, seed=1)
        assert r.degree == table3[mk][0], mk
        assert r.components == 1 and r.ties == 0
        assert r.candidates == r.total_candidates == math.comb(r.N, r.K)


def test_lifting_invariance_gpu():
    A, b = W.master_space_system(2, 4)
    degs = {B.degree(A, b, seed=s).degree for s in (1, 2, 3)}
    assert degs == {584}
    sing = {B.degree(A, b, seed=s).singular for s in (1, 2, 3)}
    assert len(sing) == 1


def test_degenerate_user_lifting_raises():
    V, _ = W.c5_points(4, n_points=10, dim=3)
    with pytest.raises(B.BdegError) as ei:
        B.degree_points(V, [7] * 10)
    assert ei.value.status == 3
    # the same through a range call reports the ties instead
    r = B.Plan.from_points(V, [7] * 10).degree_range(0, math.comb(10, 4))
    assert r.ties == enumerate_lifted(4, V, [7] * 10)["ties"] > 0


def test_generated_lifting_relifts():
    # 1-bit generated liftings are degenerate; the library re-lifts with
    # derived seeds until the subdivision is regular
    A, b = W.master_space_system(2, 2)
    r = B.degree(A, b, seed=3, lift_bits=2)
    assert r.degree == 14
    assert r.relifts >= 0 and r.ties == 0


def test_errors_and_degenerate_dimensions():
    with pytest.raises(B.BdegError) as ei:
        B.degree([[1, 1], [0, 0]], [1, 2])
    assert ei.value.status == 2
    r = B.degree([[2, 0], [0, 3]])
    assert r.dim == 0 and r.degree == 1 and r.components == 6
    # K = 1 and K = N edge cases
    V = [(3,), (1,), (2,), (5,)]
    w = [4, 9, 1, 7]
    _assert_same(_gpu(B.degree_points(V, w)), enumerate_lifted(1, V, w))
    V, w = W.c5_points(9, n_points=6, dim=5)
    _assert_same(_gpu(B.degree_points(V, w)), enumerate_lifted(6, V, w))


def test_torch_workspace_and_stream():
    A, b = W.master_space_system(2, 3)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan = B.Plan.from_system(A, b, seed=1)
        ws = plan.use_torch_workspace()
        assert ws is not None and ws.is_cuda
        r = plan.degree()
    assert r.degree == 92


def test_partial_shards_sum_to_full():
    # what each rank of a world-4 job computes, summed on one GPU
    V, w = W.c5_points(2, n_points=36, dim=5)
    full = B.Plan.from_points(V, w).degree()
    tot = [0] * B.NSLOTS
    for rank in range(4):
        plan = B.Plan.from_points(V, w, rank=rank, world=4)
        slots = torch.zeros(B.NSLOTS, dtype=torch.int64, device="cuda")
        plan.degree_partial(slots.data_ptr())
        torch.cuda.synchronize()
        for i, v in enumerate(slots.cpu().tolist()):
            tot[i] += v
    r = B.Plan.from_points(V, w).finalize(tot)
    assert (r.degree, r.cells, r.singular, r.candidates) == (full.degree, full.cells, full.singular, full.candidates)


@pytest.mark.slow
def test_w34_w26_full():
    # 3.8e9 candidates each (Table 3: 26762 and 22304)
    for mk, want in [((3, 4), 26762), ((2, 6), 22304)]:
        A, b = W.master_space_system(*mk)
        assert B.degree(A, b, seed=1).degree == want


@pytest.mark.parametrize("name", ["W2_3", "W3_2", "dp0", "rnc7"])
def test_degree_only_mode(name):
    # skipping cell-dead subtrees (P:913-929 monotonicity) keeps degree, cells,
    # candidates and ties exact; the singular count becomes an upper bound (skipped
    # subtrees count as singular: the kernel counts non-singular candidates)
    A, b = W.named_system(name)
    lift = W.liftings(len(A) + 1, 1)
    full = B.Plan.from_system(A, b, lift).degree()
    fast = B.Plan.from_system(A, b, lift, flags=0x40).degree()
    assert (fast.degree, fast.cells, fast.candidates, fast.ties) == (full.degree, full.cells, full.candidates, full.ties)
    assert fast.singular >= full.singular and not fast.singular_complete and full.singular_complete


def test_degree_only_table3(table3):
    for mk in [(2, 4), (3, 3), (2, 5)]:
        A, b = W.master_space_system(*mk)
        r = B.degree(A, b, seed=1, flags=0x40)
        assert r.degree == table3[mk][0] and r.candidates == r.total_candidates


def test_cell_emission_matches_oracle():
    # the emitted cells (index sets and NVol) are the oracle's
    from oracle import cell_list
    for (V, w, K) in [(W.c5_points(1, n_points=14, dim=4) + (5,)),
                      (W.c5_points(3, n_points=24, dim=3) + (4,))]:
        plan = B.Plan.from_points(V, w)
        assert plan.cells() == cell_list(K, V, w)
    A, b = W.master_space_system(2, 2)
    lift = W.liftings(len(A) + 1, 1)
    K, V, w = point_configuration(A, b, lift)["cone"]
    got = B.Plan.from_system(A, b, lift, flags=B.bdeg.FLAG_NATURAL_ORDER).cells()
    assert got == cell_list(K, V, w) and len(got) == 14
    plan = B.Plan.from_system(A, b, lift)              # default order: masks refer to plan.points()
    Kp, Vp, wp = plan.points()
    assert plan.cells() == cell_list(Kp, Vp, wp)


@pytest.mark.parametrize("name", ["twisted_cubic", "dp0", "W1_5", "W2_2", "W2_3", "rnc9"])
def test_walk_matches_enumeration(name):
    # walking the subdivision finds exactly the enumerated cells
    A, b = W.named_system(name)
    lift = W.liftings(len(A) + 1, 1)
    o, _ = _oracle_system(A, b, lift)
    r = B.Plan.from_system(A, b, lift).degree_walk()
    assert (r.degree, r.cells) == (o["volume"], o["cells"])


def test_walk_frontier_recollection(monkeypatch):
    # a frontier buffer too small for every growing level: the level's cells
    # are re-collected from the hash set by their level tag (same answer)
    V, w = W.c5_points(2, n_points=36, dim=5)
    base = B.Plan.from_points(V, w).degree_walk()
    monkeypatch.setenv("BDEG_WALK_TIGHT", "1")
    r = B.Plan.from_points(V, w).degree_walk()
    assert (r.degree, r.cells) == (base.degree, base.cells)
    o = enumerate_range(6, V, w, threads=8)
    assert (r.degree, r.cells) == (o["volume"], o["cells"])


def test_walk_window_eviction(monkeypatch, capfd):
    # a hash set far too small for the subdivision: levels older than L-1 are
    # dropped whenever it is rebuilt (BFS window), same degree and cells
    V, w = W.c5_points(1)
    base = B.Plan.from_points(V, w).degree_walk()
    assert (base.degree, base.cells) == (51983602, 5152)
    monkeypatch.setenv("BDEG_WALK_CAP0", "64")
    monkeypatch.setenv("BDEG_DEBUG", "1")
    r = B.Plan.from_points(V, w).degree_walk()
    err = capfd.readouterr().err
    assert (r.degree, r.cells) == (base.degree, base.cells)
    ev = int(err.split("window evictions ")[1].split(",")[0])
    assert ev >= 1, err
    monkeypatch.setenv("BDEG_WALK_TIGHT", "1")     # and with frontier re-collection on top
    r = B.Plan.from_points(V, w).degree_walk()
    assert (r.degree, r.cells) == (base.degree, base.cells)
    A, b = W.master_space_system(3, 3)
    r = B.Plan.from_system(A, b, seed=1).degree_walk()
    assert r.degree == 1620


def test_walk_narrow_storage_redo(monkeypatch, capfd):
    # tier-0 plans walk with int32 storage; a plan forced into tier 0 whose
    # minors exceed int32 (C5: lift minors ~38 bits) redoes those cells with
    # int64 storage — same degree and cells as the int64 walk and the pins
    V, w = W.c5_points(1)
    monkeypatch.setenv("BDEG_DEBUG", "1")
    r = B.Plan.from_points(V, w, flags=B.bdeg.FLAG_FORCE_TIER0).degree_walk()
    err = capfd.readouterr().err
    assert (r.degree, r.cells) == (51983602, 5152)
    assert "narrow 1" in err and int(err.split("int64 redo ")[1].split(")")[0]) > 0, err
    for mk in [(2, 4), (3, 3)]:                 # master space: tier 0, nothing redone
        A, b = W.master_space_system(*mk)
        r = B.Plan.from_system(A, b, seed=1).degree_walk()
        err = capfd.readouterr().err
        assert "narrow 1 (int64 redo 0)" in err, err
        monkeypatch.setenv("BDEG_WALK_WIDE", "1")
        r2 = B.Plan.from_system(A, b, seed=1).degree_walk()
        monkeypatch.delenv("BDEG_WALK_WIDE")
        assert (r.degree, r.cells) == (r2.degree, r2.cells)
        assert "narrow 0" in capfd.readouterr().err


def test_walk_points_and_c2():
    for (V, w, K) in [(W.c5_points(1, n_points=14, dim=4) + (5,)),
                      (W.c5_points(2, n_points=36, dim=5) + (6,)),
                      (W.c5_points(3, n_points=64, dim=3) + (4,))]:
        o = enumerate_range(K, V, w, threads=8)
        r = B.Plan.from_points(V, w).degree_walk()
        assert (r.degree, r.cells) == (o["volume"], o["cells"])
    for s in (5, 31):
        A, b, lift = W.c2_system(s)
        o, _ = _oracle_system(A, b, lift)
        r = B.Plan.from_system(A, b, lift).degree_walk()
        assert (r.degree, r.cells) == (o["volume"], o["cells"])


def test_walk_full_c5_and_table3(table3):
    V, w = W.c5_points(1)
    full = B.Plan.from_points(V, w).degree()
    walk = B.Plan.from_points(V, w).degree_walk()
    assert (walk.degree, walk.cells) == (full.degree, full.cells) == (51983602, 5152)
    for mk in [(2, 4), (3, 3), (2, 5), (3, 4), (2, 6)]:
        A, b = W.master_space_system(*mk)
        r = B.Plan.from_system(A, b, seed=1).degree_walk()
        assert r.degree == table3[mk][0], mk


def test_walk_degenerate_lifting():
    V, _ = W.c5_points(4, n_points=10, dim=3)
    with pytest.raises(B.BdegError) as ei:
        B.Plan.from_points(V, [7] * 10).degree_walk()
    assert ei.value.status == 3


def test_emitted_cells_with_normals_are_lower_facets():
    # f2: every emitted cell with its exact normal satisfies the lower-face
    # system I(sigma) strictly and the NVol is |det V_sigma|
    from fractions import Fraction
    from oracle.snf import det_fraction
    V, w = W.c5_points(2, n_points=30, dim=4)
    plan = B.Plan.from_points(V, w)
    cells = plan.cells()
    assert len(cells) == enumerate_range(5, V, w, threads=8)["cells"]
    for cell, vol in cells[:200]:
        h = plan.cell_normal(cell)
        for l in range(len(V)):
            r = w[l] - sum(hi * vi for hi, vi in zip(h, V[l]))
            assert (r == 0) if l in cell else (r > 0)
        assert abs(det_fraction([list(V[c]) for c in cell])) == vol


def test_maximum_K_and_empty_ranges():
    # K = 32 (33 rows: the largest subset size) on a sparse configuration with
    # small minors; empty and one-candidate rank intervals
    K = 32
    V = [tuple(1 if i == j else 0 for j in range(K)) for i in range(K)]
    V.append(tuple([1] * K))
    V.append(tuple([1 if j % 3 else -1 for j in range(K)]))
    V = [(1,) + v[1:] for v in V]
    w = W.liftings(len(V), 42)
    o = enumerate_range(K, V, w, threads=8)
    plan = B.Plan.from_points(V, w)
    _assert_same(_gpu(plan.degree_range(0, math.comb(len(V), K))), o)
    for b in (0, 7, math.comb(len(V), K)):
        r = plan.degree_range(b, b)
        assert (r.candidates, r.degree, r.cells, r.singular) == (0, 0, 0, 0)
    for b in (0, 100, math.comb(len(V), K) - 1):
        _assert_same(_gpu(plan.degree_range(b, b + 1)), enumerate_range(K, V, w, b, b + 1))


def test_front_end_at_scale_table2():
    # GPU row reduction mod primes reproduces Table 2,
    # dims up to m = k = 40 (n = 4800 variables), and Table 1 entries checked
    # against the exact SNF of the front end
    import os
    want = {}
    with open(os.path.join(os.path.dirname(__file__), "golden", "table2_dims.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                mm, dd = map(int, line.split())
                want[mm] = dd
    for mm in sorted(want):
        A, b = W.master_space_system(mm, mm)
        assert B.dimension_modp(A) == want[mm], mm
    from oracle import analyze
    for (m, k) in [(2, 3), (3, 5), (4, 7), (8, 8)]:
        A, b = W.master_space_system(m, k)
        assert B.dimension_modp(A) == analyze(A, b)["dim"]
    rng = W.SplitMix64(9)                     # random full-rank and rank-deficient matrices
    for _ in range(6):
        n, m = 3 + rng.uniform_int(0, 20), 2 + rng.uniform_int(0, 20)
        A = [[rng.uniform_int(-5, 5) for _ in range(m)] for _ in range(n)]
        if m > 2:
            for i in range(n):
                A[i][m - 1] = A[i][0] - 2 * A[i][1]
        assert B.dimension_modp(A) == analyze(A)["dim"]



def test_cells_are_delaunay_for_paraboloid_lifting():
    # The emitted cell list under the lifting w(p) = |p|^2 is
    # the Delaunay triangulation (lower faces of the lifted points),
    # checked against qhull (scipy) — independent of both the kernel and the
    # oracle — at sizes that span several work items (N up to 60).
    spatial = pytest.importorskip("scipy.spatial")
    checked = 0
    for seed in range(60):
        d = 2 + seed % 2
        n = 40 + seed % 21 if d == 2 else 24 + seed % 13
        lo, hi = (-20, 20) if d == 2 else (-8, 8)
        pts, _ = W.random_point_set(9100 + seed, d, n, lo, hi)
        pts = list(dict.fromkeys(pts))
        V = [(1,) + p for p in pts]
        w = [sum(x * x for x in p) for p in pts]
        tri = spatial.Delaunay(pts)
        if len(tri.coplanar):
            continue
        plan = B.Plan.from_points(V, w)
        try:
            r = plan.degree()
        except B.BdegError as e:
            if e.status == B.bdeg.BDEG_E_DEGENERATE:     # cospherical points: ties
                continue
            raise
        want = sorted(tuple(sorted(int(i) for i in s)) for s in tri.simplices)
        got = plan.cells()
        assert [c for c, _ in got] == want, seed
        assert r.cells == len(want) and r.ties == 0
        assert r.degree == sum(v for _, v in got)
        checked += 1
    assert checked >= 20, checked


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_auto_tier2_wide_values_match_oracle(seed):
    # planner-chosen tier 2 (int64 values, checked int128 products; DESIGN.md
    # §3) on V-minors of ~2^39 and lift minors of ~2^51, bit-exact vs the oracle
    r = random.Random(seed)
    K, N = 4, 16
    V = [(1,) + tuple(r.randint(-(1 << 12), 1 << 12) for _ in range(K - 1)) for _ in range(N)]
    w = [r.randint(0, 1 << 24) for _ in range(N)]
    plan = B.Plan.from_points(V, w)
    assert plan.info().tier == 2
    got = plan.degree()
    want = enumerate_lifted(K, V, w)
    assert (got.degree, got.cells, got.singular, got.ties) == \
        (want["volume"], want["cells"], want["singular"], want["ties"])
    from oracle import cell_list
    assert plan.cells() == cell_list(K, V, w)
