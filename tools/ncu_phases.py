#!/usr/bin/env python
"""Instructions and stall samples per kernel phase from an ncu report's source page.
usage: ncu_phases.py rep.ncu-rep n_elements file.cu  start1:name1 start2:name2 ...
Lines before the first start are reported as "helpers" (inlined device functions)."""
import csv
import io
import subprocess
import sys

rep, nel, want = sys.argv[1], float(sys.argv[2]), sys.argv[3]
marks = sorted((int(a.split(":")[0]), a.split(":")[1]) for a in sys.argv[4:])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Instructions Executed" in r and r[0] == "Line No")
ie = hdr.index("Instructions Executed")
ws = next(i for i, h in enumerate(hdr) if h.startswith("Warp Stall Sampling (All"))
f = None
agg = {}
tot_i = tot_s = 0.0
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) <= max(ie, ws) or not r[0].isdigit() or r[2] != "-":
        continue
    try:
        ins = float(r[ie] or 0) * 32 / nel
        st = float(r[ws] or 0)
    except ValueError:
        continue
    tot_i += ins
    tot_s += st
    if f != want:
        name = "other:" + (f or "?")
    else:
        ln = int(r[0])
        name = "helpers"
        for s0, nm in marks:
            if ln >= s0:
                name = nm
    a = agg.setdefault(name, [0.0, 0.0])
    a[0] += ins
    a[1] += st
print(f"{'phase':28s} {'slots/elem':>10s} {'stall%':>7s}")
for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:28s} {i:10.2f} {100 * s / max(tot_s, 1):7.1f}")
print(f"{'total':28s} {tot_i:10.2f}")
