"""Print an ncu launch list (--metrics gpu__time_duration.sum --csv) as id, kernel, grid, us.

Usage: python tools/checks/launch_table.py launches.csv [first] [count]
"""
import csv
import io
import sys

lines = open(sys.argv[1]).read().splitlines()
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
count = int(sys.argv[3]) if len(sys.argv) > 3 else 10**9
head = next(k for k, line in enumerate(lines) if line.startswith('"ID"'))
total = 0.0
for r in csv.DictReader(io.StringIO("\n".join(lines[head:]))):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    i = int(r["ID"])
    if i < first or i >= first + count:
        continue
    us = float(r["Metric Value"]) / 1e3
    total += us
    print(f'{i:4d} {r["Kernel Name"].split("(")[0][:44]:44s} {r["Grid Size"]:>14s} {us:9.1f} us')
print(f"total {total:.1f} us")
