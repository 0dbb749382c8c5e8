"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv): per
kernel launches, mean duration and share of device time.

  python tools/launch_summary.py launches.csv > summary.txt
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[1:]:
    name = r[ki].split("(")[0]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
T = sum(tot.values())
print("ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised):", sys.argv[1])
for k, v in tot.most_common():
    print("%-45s launches=%4d  mean=%10.2f us  total=%11.1f us  share=%5.1f%%" % (k, cnt[k], v / cnt[k], v, 100 * v / T))
