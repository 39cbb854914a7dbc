#!/usr/bin/env python
"""Debug counters per step for a given density / window (diagnostic).
usage: MA_DEBUG_COUNTERS=1 python tools/dbg_window.py dim density m steps"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_15593_b200 as ma  # noqa: E402

d, dens, m, steps = int(float(sys.argv[1])), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
levels = int(sys.argv[5]) if len(sys.argv) > 5 else 0
L = ma.lib()
s = torch.cuda.current_stream().cuda_stream
eng = ma.MicroAdam(d, dict(density=dens, window=m), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
p = torch.empty(d, dtype=torch.bfloat16, device="cuda")
g = torch.empty(d, dtype=torch.bfloat16, device="cuda")
ma._capi.check(L.ma_fill_synthetic(p.data_ptr(), 2, d, 1, 0, 0, 0, s))
prev = None
nb = d // 4096
for i in range(steps):
    ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), 2, d, 42, i + 1, 0, levels, s))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.step(p, g, 1e-3)
    e1.record()
    torch.cuda.synchronize()
    cur = eng.debug_counters()
    if prev is not None:
        c = {k: cur[k] - prev[k] for k in cur if k != "phase_cycles"}
        print(f"step {i + 1:3d} {e0.elapsed_time(e1):7.3f} ms  dup/blk {c['dup_entries'] / nb:6.1f}  "
              f"dup-overflow {c['dup_list_overflow_blocks'] / nb:6.3f}  refine {c['threshold_refinements'] / nb:6.3f}  "
              f"misses {c['threshold_misses'] / nb:6.3f}  toolow {c['threshold_too_low'] / nb:6.3f}  exactq/blk {c['exact_quotient_elems'] / nb:6.2f}", flush=True)
    prev = cur
