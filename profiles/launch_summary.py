"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel.
usage: python profiles/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg, cnt = defaultdict(float), defaultdict(int)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        agg[name] += v
        cnt[name] += 1
tot = sum(agg.values())
print(f"{'total ms':>10s} {'launches':>8s} {'avg us':>10s} {'share':>6s}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v / 1e6:10.3f} {cnt[k]:8d} {v / cnt[k] / 1e3:10.1f} {100 * v / tot:5.1f}%  {k}")
