#!/usr/bin/env python
"""Summarise an ncu report: key counters + hottest source lines (for profiles/)."""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'smsp__inst_executed.sum',
        'smsp__sass_branch_targets_threads_divergent.sum', 'smsp__warps_eligible.avg.per_cycle_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__grid_size', 'launch__block_size',
        'launch__shared_mem_per_block_dynamic', 'sm__cycles_elapsed.avg.per_second',
        'smsp__average_warp_latency_issue_stalled.ratio']


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, top=30):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h, units, vals = rows[0], rows[1], rows[2]
    print(f"# ncu summary of {rep}")
    print("kernel:", vals[h.index("Kernel Name")])
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k:70s} {vals[i]:>20s} {units[i]}")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    hdr = src[2]
    ie, sp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in src[3:]:
        if len(r) > max(ie, sp) and r[0] != "":
            try:
                data.append((float(r[ie] or 0), float(r[sp] or 0), r[0], r[1][:110]))
            except ValueError:
                pass
    ti = sum(d[0] for d in data) or 1
    ts = sum(d[1] for d in data) or 1
    print(f"\nhottest source lines (by stall samples); total warp-inst {ti:.4g}")
    for n, s, ln, text in sorted(data, key=lambda d: -d[1])[:top]:
        print(f"  {100*n/ti:6.2f}% inst {100*s/ts:6.2f}% samples  L{ln:<5s} {text}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
