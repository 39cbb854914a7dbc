#!/usr/bin/env python
"""Summarise an ncu report (run here, no GPU): headline metrics, per-source-line
instruction/stall shares, opcode mix. Usage: python tools/ncu_summary.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_warps", "launch__block_size", "launch__grid_size",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__shared_mem_per_block_dynamic",
        "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum", "dram__cycles_active.avg.pct_of_peak_sustained_elapsed"]
out = {}
for w in want:
    if w in hdr:
        i = hdr.index(w)
        out[w] = (vals[i], units[i])
        print(f"{w:70s} {vals[i]} {units[i]}")
mix = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
h = mix[2]
ie, samp = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
lines = []
for r in mix[3:]:
    if len(r) > max(ie, samp) and r[0]:
        try:
            lines.append((float(r[ie] or 0), float(r[samp] or 0), r[0], r[1][:96]))
        except ValueError:
            pass
ti = sum(x[0] for x in lines) or 1
ts = sum(x[1] for x in lines) or 1
print(f"\n-- top source lines by stall samples (inst% samp%) total inst {ti:.3g} --")
for x in sorted(lines, key=lambda x: -x[1])[:top]:
    print(f"{100*x[0]/ti:5.1f} {100*x[1]/ts:5.1f}  L{x[2]:<5} {x[3]}")
sass = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
h = sass[1]
ie, src = h.index("Instructions Executed"), h.index("Source")
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ops, st = Counter(), Counter()
for r in sass[2:]:
    try:
        n = float(r[ie] or 0)
    except (ValueError, IndexError):
        continue
    t = r[src].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    ops[op.split(".")[0]] += n
    for c in stalls:
        try:
            st[c] += float(r[h.index(c)] or 0)
        except ValueError:
            pass
tot = sum(ops.values()) or 1
print("\n-- opcode mix --")
print(", ".join(f"{k} {100*v/tot:.1f}%" for k, v in ops.most_common(24)))
T = sum(st.values()) or 1
print("\n-- stall reasons --")
print(", ".join(f"{k[6:]} {100*v/T:.1f}%" for k, v in st.most_common(12)))
