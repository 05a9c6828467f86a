"""CPU-side checks of the C ABI (no GPU): the library loads, exports every
entry point include/bdeg.h declares, its host front end agrees with the
oracle, and device entry points fail loudly instead of falling back."""
import ctypes
import math
import os
import re

import pytest

import workloads as W
from oracle import analyze, point_configuration

import paper_1501_02237_b200 as B
from paper_1501_02237_b200 import bdeg as BB

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "bdeg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bdeg_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    names = _declared()
    assert len(names) >= 15
    lib = ctypes.CDLL(B.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(BB.EXPORTS)


def test_built_for_sm100a():
    out = os.popen(f"cuobjdump --list-elf {B.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


@pytest.mark.parametrize("mk", [(1, 2), (2, 2), (2, 3), (3, 3), (2, 4), (3, 4), (4, 4), (2, 7), (4, 5)])
def test_front_end_matches_oracle_master_space(mk):
    A, b = W.master_space_system(*mk)
    lift = W.liftings(len(A) + 1, 1)
    cfg = point_configuration(A, b, lift)
    info = B.Plan.from_system(A, b, lift).info()
    assert (info.rank, info.dim, info.components) == (cfg["rank"], cfg["dim"], cfg["components"])
    K, V, w = cfg["cone"]
    assert (info.K, info.N, info.homogeneous) == (K, len(V), True)
    assert info.total_candidates == math.comb(len(V), K)


@pytest.mark.parametrize("seed", [5, 31, 46, 66])
def test_front_end_matches_oracle_c2(seed):
    A, b, lift = W.c2_system(seed)
    cfg = point_configuration(A, b, lift)
    for flags in (0, BB.FLAG_NO_LLL):
        info = B.Plan.from_system(A, b, lift, flags=flags).info()
        assert info.components == cfg["components"] == 2
        assert (info.K, info.N, info.homogeneous) == (5, 13, False)


def test_front_end_other_systems():
    for sysf in [W.twisted_cubic_system(), W.conifold_system(), W.dp0_system(), W.segre_system(2, 3),
                 W.veronese_system(2, 3), W.rnc_system(9)]:
        A, b = sysf
        cfg = point_configuration(A, b, W.liftings(len(A) + 1, 1))
        info = B.Plan.from_system(A, b).info()
        assert (info.dim, info.components) == (cfg["dim"], cfg["components"])
        K, V, _ = cfg["cone"]
        assert (info.K, info.N) == (K, len(V))


def test_no_homog_shortcut_flag():
    A, b = W.master_space_system(2, 2)
    info = B.Plan.from_system(A, b, flags=BB.FLAG_NO_HOMOG_SHORTCUT).info()
    assert (info.K, info.N, info.homogeneous) == (7, 13, False)


def test_inconsistent_and_dimension_zero():
    with pytest.raises(B.BdegError) as ei:
        B.Plan.from_system([[1, 1], [0, 0]], [1, 2])
    assert ei.value.status == BB.BDEG_E_INCONSISTENT
    r = B.degree([[2, 0], [0, 3]])          # d = 0: no device work
    assert (r.dim, r.degree, r.components) == (0, 1, 6)
    assert analyze([[2, 0], [0, 3]])["components"] == 6


def test_limits_and_bad_args():
    V, w = W.c5_points(1, n_points=40, dim=7)
    with pytest.raises(B.BdegError) as ei:
        B.Plan.from_points([(1,) + (0,) * 40] * 41, None)      # K = 41 > 32
    assert ei.value.status == BB.BDEG_E_TOO_LARGE
    with pytest.raises(B.BdegError) as ei:
        B.Plan.from_points(V[:5], w[:5])                          # N < K
    assert ei.value.status == BB.BDEG_E_INVALID


def test_items_partition_rank_space():
    for (V, w, K) in [(W.c5_points(1)[0], W.c5_points(1)[1], 8),
                      (W.c5_points(2, n_points=20, dim=3)[0], None, 4)]:
        p = B.Plan.from_points(V, w)
        n = p.num_items()
        rs = sorted(p.item_range(i) for i in range(n))
        assert rs[0][0] == 0 and rs[-1][1] == math.comb(len(V), K)
        assert all(rs[i][1] == rs[i + 1][0] for i in range(n - 1))
        shards = [set(p.shard_items(r, 3)) for r in range(3)]
        assert set().union(*shards) == set(range(n)) and sum(map(len, shards)) == n


def test_device_calls_fail_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    A, b = W.master_space_system(2, 2)
    with pytest.raises(B.BdegError) as ei:
        B.degree(A, b)
    assert ei.value.status == BB.BDEG_E_CUDA


def test_finalize_exact_limbs():
    from paper_1501_02237_b200.multi import pack_slots
    p = B.Plan.from_points(*W.c5_points(1, n_points=12, dim=3))
    big = (1 << 100) + 12345678901234567
    r = p.finalize(pack_slots(big, 7, 8, 9))
    assert (r.degree, r.cells, r.singular, r.candidates) == (big, 7, 8, 9)
    # limbs summed across ranks without carries (a limb slot may exceed 2^32)
    s1 = pack_slots((1 << 40) - 1, 1, 0, 5)
    s2 = pack_slots((1 << 40) - 1, 2, 0, 6)
    tot = [a + b for a, b in zip(s1, s2)]
    assert p.finalize(tot).degree == 2 * ((1 << 40) - 1)


def test_big_configuration_plans_walk_only():
    # N > 64 (W_{3,8}: N = 72, K = 26; Table 3's ">=" entries): the planner
    # accepts it for the cell walk, the rank-space entry points refuse
    A, b = W.master_space_system(3, 8)
    p = B.Plan.from_system(A, b, seed=1)
    info = p.info()
    assert (info.K, info.N) == (26, 72) and info.total_candidates == 0
    for call in (p.degree, lambda: p.degree_range(0, 10), lambda: p.cells(0, 10)):
        with pytest.raises(B.BdegError) as ei:
            call()
        assert ei.value.status == BB.BDEG_E_TOO_LARGE
    # a user lifting cannot seed the walk's start cell for N > 64
    q = B.Plan.from_system(A, b, lifting=W.liftings(len(A) + 1, 2))
    with pytest.raises(B.BdegError):
        q.degree_walk()


def test_cell_normal_matches_oracle_solve():
    # bdeg_cell_normal: h with h . v_c = omega_c on the cell, exact
    from oracle.subdivision import _solve, colex_unrank
    V, w = W.c5_points(1, n_points=14, dim=4)
    p = B.Plan.from_points(V, w)
    rng = W.SplitMix64(5)
    done = 0
    for _ in range(40):
        cell = colex_unrank(rng.uniform_int(0, math.comb(14, 5) - 1), 5)
        det, h = _solve([list(V[c]) for c in cell], [w[c] for c in cell])
        if det == 0:
            with pytest.raises(B.BdegError):
                p.cell_normal(cell)
            continue
        assert p.cell_normal(cell) == h
        done += 1
    assert done > 20


def test_planner_tier_follows_value_sizes():
    # host planner (DESIGN.md §3 "Arithmetic tiers"): sampled elimination
    # values of <= 28 bits start in tier 0, a wide lift row with narrow V rows
    # in tier 1, and V coordinates ~2^20 with a 2^50 lifting (products beyond
    # int64: the sampler's int128 retry) in tier 2
    import random

    def tier(K, N, cv, lw, seed=1):
        r = random.Random(seed)
        V = [(1,) + tuple(r.randint(-cv, cv) for _ in range(K - 1)) for _ in range(N)]
        w = [r.randint(0, lw) for _ in range(N)]
        with B.Plan.from_points(V, w) as p:
            return p.info().tier

    assert tier(4, 12, 2, 1 << 10) == 0
    assert tier(4, 12, 2, 1 << 40) == 1
    assert tier(6, 14, 1 << 12, 1 << 30) == 2
    # V coordinates ~2^20 with a 2^50 lifting: lifted minors reach ~2^150,
    # beyond the int128 tier; Hadamard's bound rejects the plan up front
    with pytest.raises(B.BdegError) as ei:
        tier(6, 14, 1 << 20, 1 << 50)
    assert ei.value.status == B.bdeg.BDEG_E_TOO_LARGE and "Hadamard" in str(ei.value)


def _warp_share(total, world, K, N, sms=148):
    # the planner's assumption on a host without a GPU: 148 SMs, resident
    # warps = 4 per CTA x min(4 CTAs (launch bounds), CTAs that fit in 228 KB
    # of shared memory with k_enumerate's layout)
    npl = 2 if N > 32 else 1
    smem = ((K + 1) * N * 8 + 15) // 16 * 16 + 65 * 34 * 8 + 4 * 16 * 8 + 16 + 4 * (K + 1) * 32 * npl * 8
    ctas = min(4, max(1, (228 * 1024) // (smem + 1024)))
    return total / (world * sms * 4 * ctas)


@pytest.mark.parametrize("name", ["c5", "w26", "w27"])
def test_work_queue_balance_at_world8(name):
    """at world = 8 no work item exceeds a quarter of a warp's
    share (items split one or more levels deeper), the queue is largest-first,
    the static prefix holds ~80% of the candidates and the items still
    partition the rank space (checked exhaustively for C5)."""
    import bench
    wl = bench.Workload(name)
    plan = wl.plan(world=8, rank=3, device=0)
    info = plan.info()
    total = math.comb(info.N, info.K)
    q = plan.queue_info()
    share = _warp_share(total, 8, info.K, info.N)
    sizes = {}
    probe = {0, max(0, q["n_split"] - 1), q["n_split"], q["n_items"] - 1, q["n_static"] - 1}
    for pos in probe:
        if 0 <= pos < q["n_items"]:
            b, e = plan.item_range(pos)
            sizes[pos] = e - b
    # the largest item is either the first split item or the first grouped one
    biggest = max(sizes[0], sizes.get(q["n_split"], 0))
    assert biggest <= share / 4, (name, biggest, share)
    assert q["n_split"] > 0 or name == "w27"
    if q["n_split"] > 0:
        assert sizes[0] >= sizes[q["n_split"] - 1]            # split part sorted by size
    # static prefix ~80% of the candidates: the interleave balances it
    assert 0 < q["n_static"] <= q["n_items"] and q["grab"] >= 1
    if name == "c5":
        covered, ivs = 0, []
        for pos in range(q["n_items"]):
            b, e = plan.item_range(pos)
            ivs.append((b, e))
        ivs.sort()
        assert ivs[0][0] == 0 and ivs[-1][1] == total
        assert all(ivs[i][1] == ivs[i + 1][0] for i in range(len(ivs) - 1))
        stat = sum(e - b for (b, e) in (plan.item_range(p) for p in range(q["n_static"])))
        assert 0.75 * total <= stat <= 0.85 * total
    # one GPU keeps the base depth (no split items): largest-first by group
    q1 = wl.plan(world=1, device=0).queue_info()
    assert q1["n_split"] == 0 and q1["n_static"] == q1["n_items"]
