#!/usr/bin/env python
"""Summarise an ncu launch list taken with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
(per-kernel launches, time, share, DRAM GB/s): python tools/launch_summary.py launches.csv"""
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_launches import kname  # noqa: E402

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "byte": 1.0,
         "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per, names = collections.defaultdict(dict), {}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    names[r[ii]] = kname(r[ki])
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
T = 0.0
for i, m in per.items():
    t = m.get("gpu__time_duration.sum", 0.0)
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    e = tot[names[i]]
    e[0] += 1
    e[1] += t
    e[2] += b
    T += t
print("total %.0f us over %d launches (ncu: cold-cache, serialised)" % (T, len(per)))
for n, (c, t, b) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print("%-40s %5d %10.1f us %6.2f%%  %7.0f GB/s" % (n[:40], c, t, 100 * t / T, b / t / 1e3 if t else 0))
