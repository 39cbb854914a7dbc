#!/usr/bin/env python
"""Step time + lean-kernel debug counters per (density, window) point (diagnostic).
Usage: python tools/sweep_counters.py [dim] density:window ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_15593_b200 as ma  # noqa: E402

d = int(float(sys.argv[1]))
d -= d % 4096
nb = d // 4096
L = ma.lib()
s = torch.cuda.current_stream().cuda_stream
dbg = os.environ.get("MA_DEBUG_COUNTERS") == "1"
for pt in sys.argv[2:]:
    dens, win = pt.split(":")
    dens, win = float(dens), int(win)
    eng = ma.MicroAdam(d, dict(density=dens, window=win), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
    p = torch.empty(d, dtype=torch.bfloat16, device="cuda")
    g = torch.empty(d, dtype=torch.bfloat16, device="cuda")
    ma._capi.check(L.ma_fill_synthetic(p.data_ptr(), 2, d, 1, 0, 0, 0, s))
    times, prev = [], None
    for i in range(win + 6):
        ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), 2, d, 42, i + 1, 0, 0, s))
        if dbg and i == win:
            eng.synchronize()
            prev = eng.debug_counters()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.step(p, g, 1e-3)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    st = sorted(times[win:])
    c = ""
    if dbg:
        cur = eng.debug_counters()
        n = (win + 6 - win) * nb
        c = {k: round((cur[k] - prev[k]) / n, 3) for k in cur if k != "phase_cycles"}
        ph = [a - b for a, b in zip(cur["phase_cycles"][:8], prev["phase_cycles"][:8])]
        if sum(ph):
            names = ["prologue", "pass1", "select", "window", "pass2", "mark", "unique", "dup"]
            c["phase_pct"] = {k: round(100 * v / sum(ph), 1) for k, v in zip(names, ph)}
    print(f"density {dens} m {win}: {st[len(st) // 2]:.3f} ms/step ({d / st[len(st) // 2] / 1e6:.2f} Gparam/s) "
          f"per block-step: {c}", flush=True)
    del eng, p, g
    torch.cuda.empty_cache()
