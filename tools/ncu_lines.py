#!/usr/bin/env python
"""Per-source-line issue slots per element from an ncu report (run here).
usage: ncu_lines.py rep.ncu-rep n_elements [file [min]]"""
import csv
import io
import subprocess
import sys

rep, nel = sys.argv[1], float(sys.argv[2])
want = sys.argv[3] if len(sys.argv) > 3 else "ma_fast.cu"
mn = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[2]
ie = h.index("Instructions Executed")
f = None
tot = 0.0
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
    if len(r) > ie and r[0] and r[0].isdigit():
        try:
            v = float(r[ie] or 0) * 32 / nel
        except ValueError:
            continue
        tot += v
        if f == want and v >= mn:
            print(f"{v:6.2f}  L{r[0]:<5} {r[1][:100]}")
print(f"total issue slots per element: {tot:.1f}")
