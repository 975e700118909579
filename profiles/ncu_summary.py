"""Summarise an ncu report: key SOL / occupancy / divergence metrics and the
hottest source lines by warp-stall samples.

usage: python profiles/ncu_summary.py report.ncu-rep [top_lines]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
KEYS = ["Duration", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Avg. Not Predicated Off Threads Per Warp", "Branch Efficiency", "Executed Ipc Active",
        "Issue Slots Busy", "Local Memory Spilling Requests"]


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
if rows:
    hdr = rows[0]
    ni, ui, vi = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    for r in rows[1:]:
        if len(r) > vi and r[ni] in KEYS:
            print(f"{r[ni]:45s} {r[vi]:>12s} {r[ui]}")
rr = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
want = ["dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__sass_average_branch_targets_threads_uniform.pct",
        "l1tex__average_t_sectors_per_request_pipe_lsu_mem_global_op_ld.ratio",
        "lts__t_sector_hit_rate.pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]
if len(rr) > 2:
    h = rr[0]
    for w in want:
        if w in h:
            print(f"{w:70s} {rr[2][h.index(w)]:>14s} {rr[1][h.index(w)]}")
sr = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "cuda,sass"))))
data = []
fname, h = "?", None
for r in sr:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        continue
    if h is None:
        continue
    try:
        w = float(r[h.index("Warp Stall Sampling (All Samples)")] or 0)
        ins = float(r[h.index("Instructions Executed")] or 0)
    except Exception:
        continue
    data.append((w, ins, fname, r[0], r[1]))
tot = sum(d[0] for d in data) or 1
toti = sum(d[1] for d in data) or 1
data.sort(key=lambda x: -x[0])
print(f"\nhottest source lines: % warp-stall samples, % warp instructions executed")
for w, ins, f, ln, s in data[:top]:
    print(f"{100 * w / tot:5.1f}% {100 * ins / toti:5.1f}%  {f}:{ln:<5s} {s.strip()[:100]}")


def region_report(data, regions):
    """regions: list of (name, file, lo, hi)."""
    tot = sum(d[0] for d in data) or 1
    toti = sum(d[1] for d in data) or 1
    acc = {}
    for w, ins, f, ln, s in data:
        try:
            ln = int(ln)
        except ValueError:
            continue
        for name, rf, lo, hi in regions:
            if f == rf and lo <= ln <= hi:
                a = acc.setdefault(name, [0.0, 0.0])
                a[0] += w
                a[1] += ins
                break
    print("\nregion                         stall%   inst%")
    for name, (w, ins) in sorted(acc.items(), key=lambda x: -x[1][0]):
        print(f"{name:30s} {100 * w / tot:6.1f} {100 * ins / toti:6.1f}")


if len(sys.argv) > 3:
    import json

    region_report(data, json.loads(open(sys.argv[3]).read()))
