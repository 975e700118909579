"""Executed warp-instructions and stall samples grouped by function region.

usage: python profiles/inst_regions.py REPORT.ncu-rep
Regions are source-line ranges of the kernel headers (kept in sync by hand).
"""
import csv, io, re, subprocess, sys
from collections import defaultdict
from pathlib import Path

CSRC = Path(__file__).resolve().parent.parent / "paper_2509_07782_b200" / "csrc"


def functions(fname):
    """(start_line, name) of each top-level function / lambda-free definition."""
    out = []
    for i, line in enumerate((CSRC / fname).read_text().splitlines(), 1):
        m = re.match(r"^(?:template <[^>]*>\s*)?(?:static\s+)?(?:__device__|__global__|__host__)"
                     r"[^(]*?\b(\w+)\s*\(", line)
        if m:
            out.append((i, m.group(1)))
        m = re.match(r"^\s+__device__ (?:void|float|bool) (\w+)\(", line)
        if m:
            out.append((i, m.group(1)))
    return sorted(out)


def region(fname, ln, cache={}):
    if fname not in cache:
        try:
            cache[fname] = functions(fname)
        except OSError:
            cache[fname] = []
    name = fname
    for start, fn in cache[fname]:
        if start <= ln:
            name = f"{fname}:{fn}"
    return name


rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
fname, h = "?", None
inst, samp = defaultdict(float), defaultdict(float)
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        continue
    if h is None or r[0] in ("", "Function Name"):
        continue
    try:
        ln = int(r[0])
        ex = float(r[h.index("Instructions Executed")] or 0)
        w = float(r[h.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    k = region(fname, ln)
    inst[k] += ex
    samp[k] += w
ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
print(f"total warp-instructions {ti:.4g}")
for k in sorted(inst, key=lambda k: -inst[k])[:25]:
    print(f"{100 * inst[k] / ti:6.1f}% inst  {100 * samp[k] / ts:6.1f}% samples  {k}")
