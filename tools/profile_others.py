#!/usr/bin/env python
"""Drive the non-default kernel families once each (for ncu captures; never a
bench number): global Top-K mode (ma_global.cu), the sparse-propagation phases
(lean kernel PH = 1 / 2), and the generic kernel (lossless EF). Usage:
    python tools/profile_others.py {global|sparse|generic} [dim]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_15593_b200 as ma  # noqa: E402

mode = sys.argv[1]
d = int(float(sys.argv[2])) if len(sys.argv) > 2 else 110_000_000
if mode == "sparse":
    d -= d % 4096  # the split step needs whole blocks
L = ma.lib()
s = torch.cuda.current_stream().cuda_stream
if mode == "global":
    eng = ma.MicroAdam(d, dict(), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16", blockwise=False)
elif mode == "generic":
    eng = ma.MicroAdam(d, dict(), param_dtype="f32", grad_dtype="f32", value_dtype="bf16")
    os.environ.pop("MA_FORCE_GENERIC", None)
else:
    eng = ma.MicroAdam(d, dict(), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
dt = {"generic": torch.float32}.get(mode, torch.bfloat16)
code = 1 if dt == torch.float32 else 2
p = torch.empty(d, dtype=dt, device="cuda")
g = torch.empty(d, dtype=dt, device="cuda")
ma._capi.check(L.ma_fill_synthetic(p.data_ptr(), code, d, 1, 0, 0, 0, s))
nb = d // 4096
stage = eng.stage_buffers(nb) if mode == "sparse" else None
for i in range(12):
    ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), code, d, 42, i + 1, 0, 0, s))
    if mode == "sparse":
        eng.step_front(g, 0, nb, stage)
        eng.step_stats(p, 1e-3)
    else:
        eng.step(p, g, 1e-3)
eng.synchronize()
print("ok", mode, eng.kernel_launches())
