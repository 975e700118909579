"""Per-kernel HBM throughput / divergence table from an ncu --metrics --csv
launch log (the rebuild, sort, loss and Adam kernels of a training step):

    python profiles/aux_summary.py profiles/r04_aux_kernels_c4.csv

GB/s = (dram__bytes_read.sum + dram__bytes_write.sum) / gpu__time_duration.sum
per launch (ncu serialises launches with cold caches: a ceiling on traffic,
a floor on speed)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, mi, ui, vi, idi = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit",
                                            "Metric Value", "ID"))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3,
         "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
per, names = collections.defaultdict(dict), {}
for r in rows[hi + 1:]:
    if len(r) <= vi or r[vi] in ("", "n/a"):
        continue
    v = float(r[vi].replace(",", ""))
    if r[mi].startswith("dram__bytes") or r[mi] == "gpu__time_duration.sum":
        v *= SCALE.get(r[ui], 1)
    per[r[idi]][r[mi]] = v
    names[r[idi]] = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for i, d in per.items():
    for m, v in d.items():
        agg[names[i]][m].append(v)
print(f"{'kernel':28s} {'n':>4s} {'avg us':>9s} {'MB/launch':>10s} {'GB/s':>8s} {'dram%':>6s} "
      f"{'sm%':>6s} {'br.eff%':>7s} {'thr/warp':>8s}")
for k, d in sorted(agg.items(), key=lambda x: -sum(x[1]["gpu__time_duration.sum"])):
    n = len(d["gpu__time_duration.sum"])
    avg = lambda m: sum(d[m]) / n  # noqa: E731
    t = avg("gpu__time_duration.sum")
    b = avg("dram__bytes_read.sum") + avg("dram__bytes_write.sum")
    print(f"{k[:28]:28s} {n:4d} {t:9.1f} {b / 1e6:10.2f} {b / (t * 1e-6) / 1e9:8.0f} "
          f"{avg('dram__throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
          f"{avg('sm__throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
          f"{avg('smsp__sass_average_branch_targets_threads_uniform.pct'):7.1f} "
          f"{avg('smsp__thread_inst_executed_per_inst_executed.ratio'):8.1f}")
