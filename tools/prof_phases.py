#!/usr/bin/env python
"""Per-phase warp-cycle shares of the lean kernel (needs an MA_LEAN_PROF=1 build via MA_LIB_PATH
and MA_DEBUG_COUNTERS=1). Diagnostic only; clock64 marks perturb timing slightly."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_15593_b200 as ma  # noqa: E402

NAMES = ["prologue", "pass1", "select", "window", "pass2", "stats-mark", "stats-unique", "stats-dup"]
d = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_100_000_000
steps = int(os.environ.get("SCAN_STEPS", "16"))
cyc = int(os.environ.get("SCAN_CYCLE", "8"))
L = ma.lib()
s = torch.cuda.current_stream().cuda_stream
eng = ma.MicroAdam(d, dict(), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
p = torch.empty(d, dtype=torch.bfloat16, device="cuda")
g = torch.empty(d, dtype=torch.bfloat16, device="cuda")
ma._capi.check(L.ma_fill_synthetic(p.data_ptr(), 2, d, 1, 0, 0, 0, s))
prev = None
for i in range(steps):
    ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), 2, d, 42, (i % cyc) + 1, 0, 0, s))
    eng.step(p, g, 1e-3)
    cur = eng.debug_counters()
    ph = cur["phase_cycles"][:8]
    if prev is not None:
        dph = [a - b for a, b in zip(ph, prev)]
        tot = sum(dph) or 1
        print(f"step {i + 1:2d}: " + "  ".join(f"{n} {100 * c / tot:5.1f}%" for n, c in zip(NAMES, dph)),
              f" cyc/blk {tot / (d // 4096):9.0f}", flush=True)
    prev = ph
