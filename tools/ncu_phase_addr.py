#!/usr/bin/env python
"""Thread-instructions per element by kernel phase from an ncu source CSV
(--print-source cuda,sass), attributing inlined helper code to the phase of
the surrounding kernel lines in SASS address order (run here, no GPU).
usage: ncu_phase_addr.py src.csv[.gz] n_elements file.cu kernel_first_line name:line ..."""
import bisect
import csv
import gzip
import io
import sys

path, nel, fname, kfirst = sys.argv[1], float(sys.argv[2]), sys.argv[3], int(sys.argv[4])
marks = sorted((int(a.split(":")[1]), a.split(":")[0]) for a in sys.argv[5:])
txt = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
rows, f, line, hdr = [], None, None, None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie, ws = r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None:
        continue
    if r[0].isdigit():
        line = (f, int(r[0]))
    elif len(r) > 3 and r[2].startswith("0x"):
        try:
            ex = float(r[ie] or 0)
        except ValueError:
            ex = 0.0
        try:
            st = float(r[ws] or 0)
        except ValueError:
            st = 0.0
        rows.append((int(r[2], 16), ex, st, line))
rows.sort()
seen, agg, cur = set(), {}, "prologue"
keys = [m[0] for m in marks]
tot = stot = 0.0
for a, ex, st, ln in rows:
    if a in seen:
        continue
    seen.add(a)
    if ln and ln[0] == fname and ln[1] >= kfirst:
        i = bisect.bisect_right(keys, ln[1]) - 1
        cur = marks[i][1] if i >= 0 else "prologue"
    v = agg.setdefault(cur, [0.0, 0.0])
    v[0] += ex * 32 / nel
    v[1] += st
    tot += ex * 32 / nel
    stot += st
for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:16s} {i:7.2f} thread-instr/elem  {100 * s / max(stot, 1):5.1f}% stall samples")
print(f"{'total':16s} {tot:7.2f}")
