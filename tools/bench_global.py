#!/usr/bin/env python
"""Wall time per step of the global Top-K mode (blockwise=false, ma_global.cu).
The step synchronises with the host between radix passes, so wall clock around
synchronous steps is the honest measure. Usage: python tools/bench_global.py [dim ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_15593_b200 as ma  # noqa: E402

L = ma.lib()
for arg in sys.argv[1:] or ["1.1e8"]:
    d = int(float(arg))
    s = torch.cuda.current_stream().cuda_stream
    eng = ma.MicroAdam(d, dict(), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16", blockwise=False)
    p = torch.empty(d, dtype=torch.bfloat16, device="cuda")
    gs = [torch.empty(d, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
    ma._capi.check(L.ma_fill_synthetic(p.data_ptr(), 2, d, 1, 0, 0, 0, s))
    for i, g in enumerate(gs):
        ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), 2, d, 42, i + 1, 0, 0, s))
    for i in range(12):  # fill the window
        eng.step(p, gs[i % 4], 1e-3)
    torch.cuda.synchronize()
    n = 10
    t = time.perf_counter()
    for i in range(n):
        eng.step(p, gs[i % 4], 1e-3)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / n * 1e3
    print(f"global d={d:,} {ms:.3f} ms/step {d / ms * 1e3:.3e} params/s", flush=True)
    del eng, p, gs
    torch.cuda.empty_cache()
