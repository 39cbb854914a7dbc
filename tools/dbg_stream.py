#!/usr/bin/env python
"""Per-step debug counters of the default step kernel on the bench's gradient
stream (bench.grad_source). usage: python tools/dbg_stream.py [dim] [steps] [mode]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MA_DEBUG_COUNTERS"] = "1"
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_15593_b200 as ma  # noqa: E402

d = int(float(sys.argv[1])) if len(sys.argv) > 1 else 110_000_000
d -= d % 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 14
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
L = ma.lib()
s = torch.cuda.current_stream().cuda_stream
eng = ma.MicroAdam(d, dict(), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
p = torch.empty(d, dtype=torch.bfloat16, device="cuda")
g = torch.empty(d, dtype=torch.bfloat16, device="cuda")
ma._capi.check(L.ma_fill_synthetic(p.data_ptr(), 2, d, 1, 0, 0, 0, s))
prev = None
nb = d // 4096
for i in range(steps):
    j, off = bench.grad_source(i, 8)
    ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), 2, d, 42, j, off, mode, s))
    eng.step(p, g, 1e-3)
    eng.synchronize()
    c = eng.debug_counters()
    c.pop("phase_cycles", None)
    if prev is not None:
        print(f"step {i + 1}: " + ", ".join(f"{k}={(c[k] - prev[k]) / nb:.4f}" for k in c), flush=True)
    prev = c
