"""Per-kernel share of a full solve from an ncu launch list (gpu__time_duration.sum CSV).

python tools/checks/kernel_mix.py launches.csv   -- kernels sorted by total time
"""
import csv
import sys
from collections import defaultdict

tot, cnt = defaultdict(float), defaultdict(int)
with open(sys.argv[1]) as f:
    rows = [r for r in csv.reader(f) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r[ui]]
    name = r[ki].split("(")[0].split("<")[0]
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
print(f"total {s / 1e3:.2f} ms over {sum(cnt.values())} launches")
for k in sorted(tot, key=tot.get, reverse=True)[:25]:
    print(f"{tot[k] / 1e3:9.3f} ms {100 * tot[k] / s:5.1f}%  {cnt[k]:6d}  {k}")
