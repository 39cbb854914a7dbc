#!/usr/bin/env python
"""Per-kernel times from an ncu --metrics gpu__time_duration.sum --csv launch list.
Usage: python tools/launch_table.py launches.csv [last_n_launches]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            data.append((d["Kernel Name"].split("(")[0][-40:], float(d["Metric Value"]) / 1e6))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for name, t in data[-n:]:
    print(f"{t:8.3f} ms  {name}")
