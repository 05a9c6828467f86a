#!/usr/bin/env python
"""Benchmark: exact degree (normalised lattice volume) of the C5 synthetic
configuration — BASELINE.json configs[4], "k=8 over 40 lifted lattice points
(~7.7e7 candidate simplices), rank space sharded across 8xB200".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5|w<m><k>] [--degree-only]
  python bench.py --impl reference ...        # the CPU oracle arm

A step = one pass of the whole hot path over the full rank space: the
enumeration kernel (+ int64-tier replay), the exact combine (one NCCL
all-reduce of 16 int64 slots when N > 1) and the D2H read of the slots.
`value` (simplices/s) = C(N,K) / device time per step, max over ranks,
inputs resident in HBM.  `e2e` = the same metric through the C ABI with
HOST buffers (bdeg_plan_points + bdeg_degree: H2D upload of the lifted
matrix and binomial table, D2H of the result) per step.

Timing rules: W untimed warm-up steps; each timed step bracketed by CUDA
events on the launching stream; L2 flushed between steps (256 MiB write,
outside the events); barrier + synchronize around the timed region; the
clocks are sampled with nvidia-smi during it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import random
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simplices/sec and time-to-degree at 1/2/4/8 B200; % integer-pipe peak"
UNIT = "simplices/s"


class Workload:
    """A bench workload as the user hands it to the library: a lifted point
    configuration (C5, `bdeg_plan_points`) or a binomial system x^A = b
    (W_{m,k}, `bdeg_plan`: the library's own SNF / P_0 / LLL front end)."""

    def __init__(self, name):
        import workloads as W
        self.name = name
        if name == "c5":
            self.kind = "points"
            self.V, self.w = W.c5_points(1)
            self.desc = ("C5 synthetic: K=8 vectors (1,a), a uniform in [-3,3]^7, N=40 distinct points, "
                         "lifting uniform in [0,2^20) (SplitMix64 seed 1)")
            self.extra = {"seed": 1}
        elif name.startswith("w") and len(name) == 3 and name[1:].isdigit():
            self.kind = "system"
            m, k = int(name[1]), int(name[2])
            self.A, self.b = W.master_space_system(m, k)
            self.lift = W.liftings(len(self.A) + 1, 1)
            self.desc = (f"master space grad W_{{{m},{k}}} (PAPER.md Table 3): x^A = b through the "
                         f"library's front end (n={len(self.A)} variables, m={len(self.A[0])} binomials)")
            self.extra = {"m": m, "k": k, "seed": 1, "point_order": "ascending lifting residual (library default for x^A = b plans)"}
        else:
            raise SystemExit(f"unknown workload {name!r} (c5 or w<m><k>)")

    def plan(self, **opts):
        import paper_1501_02237_b200 as B
        if self.kind == "points":
            return B.Plan.from_points(self.V, self.w, **opts)
        return B.Plan.from_system(self.A, self.b, self.lift, **opts)

    def h2d_bytes(self, K, N):
        """Bytes the public call uploads per step: the lifted matrix and the binomial table."""
        return (((K + 1) * N * 8 + 15) // 16) * 16 + 65 * 34 * 8

    def oracle_points(self):
        """(K, V, w) for the CPU baseline only (the oracle's own front end)."""
        if self.kind == "points":
            return len(self.V[0]), self.V, self.w
        from oracle import point_configuration  # cpu_baseline / reference arm only
        K, V, w = point_configuration(self.A, self.b, self.lift)["cone"]
        return K, V, w


def workload_sizes(name):
    """(K, N) of a workload without the GPU library: C5 directly; W_{m,k} via the
    oracle's front end (the point count is basis-independent)."""
    wl = Workload(name)
    K, V, _ = wl.oracle_points()
    return K, len(V)


def bench_config(wl, K, N, world):
    """ONE config dict, emitted identically by both arms."""
    return {"workload": wl.desc, "K": K, "N": N, "candidates": math.comb(N, K),
            "l2": "GPU arm: L2 flushed between steps (256 MiB write outside the timed events)",
            "parallelism": f"rank space sharded over {world} GPU(s): static interleaved items, "
                           "then a cross-GPU work-stealing tail; one all-reduce of 16 int64 slots",
            **wl.extra}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"bdeg_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.f.close()

    def summary(self):
        try:
            rows = [l.strip().split(", ") for l in open(self.path) if l.strip()]
        except Exception:  # noqa: BLE001
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 4 + i and "Active" in r[4 + i]
                          and "Not" not in r[4 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(rows), "reasons": reasons}


def cpu_oracle_sample(K, V, w, budget_candidates, seed=7):
    """Time the CPU oracle (C variant, all host cores) on random rank intervals."""
    from oracle.native import enumerate_range
    total = math.comb(len(V), K)
    rng = random.Random(seed)
    n_iv = 16
    span = max(1, min(total, budget_candidates) // n_iv)
    ivs = []
    for _ in range(n_iv):
        b = rng.randrange(0, max(1, total - span))
        ivs.append((b, min(total, b + span)))
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    cand = 0
    for b, e in ivs:
        r = enumerate_range(K, V, w, b, e, threads=cores)
        cand += r["candidates"]
    dt = time.perf_counter() - t0
    return cand / dt, cores, f"{n_iv} random colex-rank intervals of {span} candidates ({cand} total) of the same workload"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = Workload(args.workload)
    K, V, w = wl.oracle_points()
    total = math.comb(len(V), K)
    # each step is a bounded sample; the whole --steps/--warmup run stays at
    # ~2.4e8 candidates (about 3 minutes of the oracle on 16 host cores)
    budget = int(min(args.ref_sample, max(2e5, 2.4e8 / (args.steps + args.warmup / 4.0))))
    for _ in range(args.warmup):
        cpu_oracle_sample(K, V, w, budget // 4, seed=1)
    vals = []
    t0 = time.perf_counter()
    sample = None
    for s in range(args.steps):
        v, cores, sample = cpu_oracle_sample(K, V, w, budget, seed=100 + s)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * wall / max(1, args.steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int128",
        "data": "synthetic",
        "config": bench_config(wl, K, len(V), args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "time_to_degree_s_extrapolated": total / value,
    }
    print(json.dumps(line), flush=True)


def algorithmic_ops_per_candidate(K, nonsingular_frac, tested=2.0):
    """SURVEY §8.d 'Algorithmic work per candidate' (integer ops, an update
    u = (a*b - c*d)/e counted as 4): Bareiss (K-1)K(2K-1)/6 updates; for
    det != 0 the lift functional (K(K+1)/2 multiply-adds = 2 ops each, plus K
    exact divisions) and the facet test (E[#tested] ~ 2 points x (K+1)
    multiply-adds).  676 at K = 8 with no singular candidates."""
    bareiss = 4.0 * (K - 1) * K * (2 * K - 1) / 6.0
    lift = K * (K + 1) + K
    facet = 2.0 * tested * (K + 1)
    return bareiss + nonsingular_frac * (lift + facet)


def load_int_peak():
    """The measured integer issue peak (tools/intpipe_bench.cu on a B200):
    lane-ops per SM clock, the best integer instruction mix (ALU + FMA pipes
    together) and the ALU pipe alone."""
    pth = os.path.join(ROOT, "profiles", "r2_intpipe_peaks.json")
    if os.path.exists(pth):
        d = json.load(open(pth))
        rows = {k: v for k, v in d.items() if isinstance(v, dict) and "lane_ops_per_clk_per_sm" in v}
        alu = max(v["lane_ops_per_clk_per_sm"] for v in rows.values() if v["pipe"] == "alu")
        allp = max(v["lane_ops_per_clk_per_sm"] for v in rows.values())
        best = max(rows, key=lambda k: rows[k]["lane_ops_per_clk_per_sm"])
        return allp, alu, f"measured, best mix '{best}' (profiles/r2_intpipe_peaks.json)"
    return 128.0, 64.0, "fallback: 4 SMSP x 32 lanes issue/clk/SM (not measured)"


def run_gpu(args):
    import torch
    import torch.distributed as dist
    import paper_1501_02237_b200 as B

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # BDEG_SHARE_GPU=1 (testing only): ranks share the visible GPUs round-robin
    # and combine over gloo, to exercise the multi-rank path on a 1-GPU box
    share = os.environ.get("BDEG_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    wl = Workload(args.workload)
    stream = torch.cuda.current_stream()
    flags = B.bdeg.FLAG_DEGREE_ONLY if args.degree_only else 0

    plan = wl.plan(rank=rank, world=world, stream=stream.cuda_stream, device=local, flags=flags)
    plan.use_torch_workspace(local)
    info = plan.info()
    K, N = info.K, info.N
    total = math.comb(N, K)
    steal = world > 1 and os.environ.get("BDEG_STEAL", "1") == "1"
    if steal:        # static share first, then one global tail queue (CUDA IPC + NVLink atomics)
        from paper_1501_02237_b200.multi import enable_work_stealing
        enable_work_stealing(plan, local)
    slots = torch.zeros(B.NSLOTS, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        plan.degree_partial(slots.data_ptr())
        if world > 1:
            dist.all_reduce(slots, op=dist.ReduceOp.SUM)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    res = plan.finalize(slots.cpu().tolist())

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = B.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        time.sleep(0.3)                                  # let nvidia-smi attach before timing
        t_wall0 = time.perf_counter()
        for s in range(args.steps):
            flush.fill_(float(s))                       # L2 flush (outside the events)
            evs[s][0].record(stream)
            step()
            evs[s][1].record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
        if world > 1:
            dist.barrier()
        time.sleep(0.05)
    launches = B.launch_count() - launches0
    ms = [a.elapsed_time(b) for a, b in evs]
    ms_step = statistics.mean(ms)
    tt = torch.tensor([ms_step], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_step = float(tt.item())
    res = plan.finalize(slots.cpu().tolist())
    value = total / (ms_step / 1000.0)

    # ---- e2e: the public C-ABI call with HOST buffers, every step (planning
    # from the host inputs incl. the front end, H2D, kernel, D2H of the slots)
    e2e_ms = []
    h2d = wl.h2d_bytes(K, N)
    d2h = B.NSLOTS * 8
    e2e_steps = min(args.steps, 30)     # a plan per step: bounded to keep the run short
    for s in range(args.warmup + e2e_steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        with wl.plan(rank=rank, world=world, stream=stream.cuda_stream, device=local, flags=flags) as p2:
            if world == 1:
                r2 = p2.degree()
            else:
                from paper_1501_02237_b200.multi import degree_distributed
                r2 = degree_distributed(p2, dev)
        dt = (time.perf_counter() - t0) * 1000.0
        if s >= args.warmup:
            e2e_ms.append(dt)
        assert r2.degree == res.degree
    e2e = torch.tensor([statistics.mean(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    e2e_step = float(e2e.item())

    if rank == 0 and world > 1:
        # the combined shards must equal a single-GPU run over the whole rank space
        with wl.plan(stream=stream.cuda_stream, device=local, flags=flags) as p1:
            full = p1.degree()
        assert (full.degree, full.cells, full.candidates) == (res.degree, res.cells, res.candidates), \
            "multi-GPU combine differs from the single-GPU result"
    if rank == 0:
        peaks, peak_kind = load_peaks()
        sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        lanes, alu_lanes, lanes_kind = load_int_peak()
        peak_ops = lanes * n_sm * sm_mhz * 1e6 * world
        t_s = ms_step / 1000.0
        # (1) SURVEY §8.d's algorithmic integer ops per candidate (the headline frac)
        nonsing = 1.0 - (res.singular / res.candidates if res.candidates and not args.degree_only else 0.0)
        opc = algorithmic_ops_per_candidate(K, nonsing)
        achieved = opc * total / t_s
        # (2) the kernel's own work (its counters): 4 ops per fraction-free
        # update + 2 per point per leaf facet test
        own_ops = 4.0 * res.updates + 2.0 * res.leaves * N
        # (3) executed instructions of the same kernel (committed ncu --set full capture)
        executed = None
        ep = os.path.join(ROOT, "profiles", "ncu_executed.json")
        if os.path.exists(ep):
            executed = json.load(open(ep)).get(args.workload)
        exec_frac = None
        if executed and executed.get("warp_inst_per_launch"):
            thr = executed["warp_inst_per_launch"] * executed.get("threads_per_inst", 32.0)
            exec_frac = thr / t_s / peak_ops
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(args.workload)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            Ko, Vo, wo = wl.oracle_points()
            v, cores, sample = cpu_oracle_sample(Ko, Vo, wo, args.ref_sample)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": B.bdeg.TIER_DTYPE[info.tier],
            "data": "synthetic",
            "config": bench_config(wl, K, N, world),
            "kernel": {"inner_levels": info.inner_levels, "tier": info.tier, "work_items": plan.num_items(),
                       "dead_subtrees_in_full_mode": info.dead_full,
                       "degree_only": bool(args.degree_only), "work_stealing_tail": steal},
            "time_to_degree_ms": e2e_step,
            "result": {"degree": res.degree, "cells": res.cells, "singular": res.singular,
                       "candidates": res.candidates, "ties": res.ties,
                       "overflow_reruns": res.overflow_reruns, "leaves": res.leaves},
            "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": peak_ops / 1e12,
                         "unit": "Tintop/s", "frac": achieved / peak_ops, "traffic": traffic,
                         "peak_basis": f"{lanes:.1f} integer lane-ops/clk/SM ({lanes_kind}) x {n_sm} SMs x "
                                       f"{sm_mhz:.0f} MHz ({peak_kind} sm_max_mhz) x {world} GPU(s)",
                         "algorithmic_ops_per_candidate": opc,
                         "fractions": {
                             "algorithmic_8d": achieved / peak_ops,
                             "own_work": own_ops / t_s / peak_ops,
                             "ncu_executed": exec_frac,
                             "alu_pipe_only_algorithmic": achieved / (alu_lanes * n_sm * sm_mhz * 1e6 * world)},
                         "ncu_executed": executed},
            "cpu_baseline": cpu,
            "e2e": {"value": total / (e2e_step / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "wall_s_timed_region": t_wall,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="bdeg", choices=["bdeg", "reference"])
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--ref-sample", type=int, default=4_000_000,
                    help="candidates per oracle sample (cpu_baseline / reference arm)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--degree-only", action="store_true",
                    help="skip cell-dead subtrees (singular becomes an upper bound)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
