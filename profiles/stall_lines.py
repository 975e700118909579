"""Per-source-line warp-stall attribution from an ncu report (cuda,sass view).

usage: python profiles/stall_lines.py REPORT.ncu-rep [stall_column] [topN]
Prints the source lines with the most samples of the given stall reason
(default: all samples) plus their share of all samples.
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "Warp Stall Sampling (All Samples)"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
import os
kf = ["--kernel-name", os.environ["KERNEL"]] if os.environ.get("KERNEL") else []  # e.g. regex:k_render_camera
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                      "--print-source", "cuda,sass", *kf],
                     capture_output=True, text=True).stdout
fname, h, data = "?", None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        continue
    if h is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        v = float(r[h.index(col)] or 0)
        w = float(r[h.index("Warp Stall Sampling (All Samples)")] or 0)
        ex = float(r[h.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    data.append((v, w, ex, fname, r[0], r[1]))
tv = sum(d[0] for d in data) or 1.0
tw = sum(d[1] for d in data) or 1.0
print(f"{col}: {tv:.0f} samples = {100 * tv / tw:.1f}% of all {tw:.0f}")
data.sort(key=lambda d: -d[0])
for v, w, ex, f, ln, s in data[:top]:
    print(f"{100 * v / tv:5.1f}%  all={100 * w / tw:5.1f}%  inst={ex:10.3g}  "
          f"{f}:{ln:<5s} {s.strip()[:70]}")
