#!/usr/bin/env python
"""Per-source-line thread-instructions per element for one kernel of an ncu
report (run here, no GPU). usage: ncu_src_lines.py rep.ncu-rep n_elements kernel_substr [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, nel, kern = sys.argv[1], float(sys.argv[2]), sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.Counter()
src = {}
f = fn = None
ie = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif r[0] == "Function Name":
        fn = r[1]
    elif r[0] == "Line No":
        ie = r.index("Instructions Executed")
    elif ie and r[0].isdigit() and len(r) > ie and kern in (fn or ""):
        try:
            v = float(r[ie] or 0) * 32 / nel
        except ValueError:
            continue
        agg[(f, int(r[0]))] += v
        src[(f, int(r[0]))] = r[1].strip()[:100]
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:6.2f} {f}:{l:<5} {src[(f, l)]}")
print(f"total thread-instructions per element in {kern}: {sum(agg.values()):.1f}")
