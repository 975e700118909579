"""Headline metrics + stall breakdown of the first kernel in an ncu report.

usage: python profiles/ncu_stalls.py REPORT.ncu-rep
"""
import csv, subprocess, sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, v = rows[0], rows[2]
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]
for k in keys:
    if k in h:
        print(f"{k:60s} {v[h.index(k)][:110]}")
print("-- stalls (warps per issue)")
st = []
for k, x in zip(h, v):
    if (k.startswith("smsp__average_warps_issue_stalled_") and
            k.endswith("_per_issue_active.ratio")):
        try:
            st.append((float(x), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
for x, k in sorted(st, reverse=True)[:10]:
    print(f"  {k:30s} {x:7.3f}")
