#!/usr/bin/env python
"""Debug counters of the lean kernel over N steps (MA_DEBUG_COUNTERS=1 build-independent).
Usage: MA_LIB_PATH=... python tools/dbg_counters.py [dim] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MA_DEBUG_COUNTERS"] = "1"
import torch  # noqa: E402

import paper_2405_15593_b200 as ma  # noqa: E402

d = int(float(sys.argv[1])) if len(sys.argv) > 1 else 110_000_000
d -= d % 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 14
L = ma.lib()
s = torch.cuda.current_stream().cuda_stream
eng = ma.MicroAdam(d, dict(), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
p = torch.empty(d, dtype=torch.bfloat16, device="cuda")
g = torch.empty(d, dtype=torch.bfloat16, device="cuda")
ma._capi.check(L.ma_fill_synthetic(p.data_ptr(), 2, d, 1, 0, 0, 0, s))
for i in range(steps):
    ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), 2, d, 42, i + 1, 0, 0, s))
    eng.step(p, g, 1e-3)
eng.synchronize()
c = eng.debug_counters()
c.pop("phase_cycles", None)
print(d // 4096, "blocks x", steps, "steps:", c)
