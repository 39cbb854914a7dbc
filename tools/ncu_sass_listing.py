#!/usr/bin/env python
"""SASS listing of one kernel from an ncu report (run here, no GPU): address,
executed warp-instructions per element-block, stall samples and source line.
usage: ncu_sass_listing.py rep.ncu-rep n_units [kernel_substr] > listing.txt
n_units scales 'Instructions Executed' (e.g. number of 4096-blocks)."""
import csv
import io
import subprocess
import sys

rep, nunits = sys.argv[1], float(sys.argv[2])
kern = sys.argv[3] if len(sys.argv) > 3 else "microadam_step_lean"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
f = fn = None
hdr = None
line = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif r[0] == "Function Name":
        fn = r[1]
    elif r[0] == "Line No":
        hdr = r
        ie = r.index("Instructions Executed")
        ws = r.index("Warp Stall Sampling (All Samples)")
    elif hdr and kern in (fn or ""):
        if r[0].isdigit():
            line = f"{f}:{r[0]}"
        elif r[2].startswith("0x"):
            rows.append((int(r[2], 16), r[3], float(r[ie] or 0), float(r[ws] or 0), line))
rows.sort()
base = rows[0][0] if rows else 0
seen = set()
for a, ins, ex, st, ln in rows:
    if a in seen:
        continue
    seen.add(a)
    print(f"{a - base:6x} {ex / nunits:8.3f} {st:6.0f}  {ins:60s} {ln}")
