#!/usr/bin/env python
"""Top source lines by warp-stall samples (all + long scoreboard) of an ncu report
or of its exported source CSV (run here). usage: ncu_stall_lines.py rep.ncu-rep|src.csv [top]"""
import collections
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
if path.endswith(".csv"):
    out = open(path).read()
else:
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


hdr = None
f = None
agg, lsb, ins, src = collections.Counter(), collections.Counter(), collections.Counter(), {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ws, ie, ls = r.index("Warp Stall Sampling (All Samples)"), r.index("Instructions Executed"), r.index("stall_long_sb")
        continue
    if hdr and r[0].isdigit():
        k = f"{f}:{r[0]}"
        src[k] = r[1][:80]
        agg[k] += num(r[ws])
        lsb[k] += num(r[ls])
        ins[k] += num(r[ie])
tot = sum(agg.values())
print(f"samples {tot:.0f}, long_scoreboard {100 * sum(lsb.values()) / tot:.1f}%")
for k, v in agg.most_common(top):
    print(f"{100 * v / tot:5.1f}% all {100 * lsb[k] / tot:5.1f}% lsb  {k:24s} {src[k]}")
