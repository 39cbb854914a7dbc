#!/usr/bin/env python
"""Top source lines (thread-instructions per element, stall share) per kernel from
an `ncu --page source --csv --print-source cuda,sass` dump (gzip ok).
Usage: python tools/ncu_src_top.py src.csv[.gz] n_elements [kernel_substr] [top]"""
import collections
import csv
import gzip
import io
import sys

path, nel = sys.argv[1], float(sys.argv[2])
sub = sys.argv[3] if len(sys.argv) > 3 else ""
top = int(sys.argv[4]) if len(sys.argv) > 4 else 12
fh = io.TextIOWrapper(gzip.open(path), "utf-8") if path.endswith(".gz") else open(path)


def fl(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


fn = fp = hdr = None
agg = collections.defaultdict(collections.Counter)
stall = collections.defaultdict(collections.Counter)
src = {}
for r in csv.reader(fh):
    if not r:
        continue
    if r[0] == "File Path":
        fp = r[1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[2] == "-" and sub in (fn or ""):
        d = dict(zip(hdr, r))
        key = (fp.split("/")[-1], int(r[0]))
        agg[fn][key] += fl(d["Thread Instructions Executed"])
        stall[fn][key] += fl(d["Warp Stall Sampling (All Samples)"])
        src[key] = r[1][:100]
for fn in agg:
    tot, st = sum(agg[fn].values()), sum(stall[fn].values()) or 1
    print(f"== {fn[:70]}  {tot / nel:.1f} thread-instr/elem")
    for k, v in sorted(agg[fn].items(), key=lambda x: -x[1])[:top]:
        print(f"  {v / nel:6.2f}/elem {100 * stall[fn][k] / st:5.1f}% stall  {k[0]}:{k[1]}  {src[k]}")
