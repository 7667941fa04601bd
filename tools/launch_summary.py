"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, average durations and shares of the summed time.
Usage: python tools/launch_summary.py launches.csv "header line" > profiles/X.txt"""
import csv
import re
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
acc = OrderedDict()
for r in rows[1:]:
    name = re.sub(r"\(.*$", "", r[ki]).replace("void ", "")
    us = float(r[vi].replace(",", "")) / 1e3
    a = acc.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(v[1] for v in acc.values())
print(sys.argv[2] if len(sys.argv) > 2 else "# ncu launch list")
print("# per-launch durations under ncu (serialised, cache-flushed): compare shares, not absolutes")
print(f"{'kernel':44s} {'launches':>8s} {'avg_us':>10s} {'total_us':>10s} {'share':>7s}")
for k, (n, t) in sorted(acc.items(), key=lambda x: -x[1][1]):
    print(f"{k[:44]:44s} {n:8d} {t / n:10.1f} {t:10.1f} {100 * t / tot:6.1f}%")
