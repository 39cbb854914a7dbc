#!/usr/bin/env python
"""Device time per step of the global Top-K mode (blockwise=false, ma_global.cu),
window full, a fresh gradient every step (filled outside the timed region).
Usage: python tools/bench_global.py [dim ...]   (MA_GLOBAL_BRACKET=0: full digit passes)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_15593_b200 as ma  # noqa: E402

L = ma.lib()
heavy = os.environ.get("GRAD_STREAM") == "heavy"
for arg in sys.argv[1:] or ["1.1e8"]:
    d = int(float(arg))
    s = torch.cuda.current_stream().cuda_stream
    eng = ma.MicroAdam(d, dict(), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16", blockwise=False)
    p = torch.empty(d, dtype=torch.bfloat16, device="cuda")
    g = torch.empty(d, dtype=torch.bfloat16, device="cuda")
    ma._capi.check(L.ma_fill_synthetic(p.data_ptr(), 2, d, 1, 0, 0, 0, s))
    times = []
    for i in range(20):
        ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), 2, d, 42, i + 1, 0, 2 if heavy else 0, s))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.step(p, g, 1e-3)
        e1.record()
        torch.cuda.synchronize()
        if i >= 10:  # window full (m = 10)
            times.append(e0.elapsed_time(e1))
    ms = sorted(times)[len(times) // 2]
    print(f"global d={d:,} {ms:.3f} ms/step (median of steps 11-20; {' '.join(f'{t:.2f}' for t in times)}) "
          f"{d / ms * 1e3:.3e} params/s", flush=True)
    del eng, p, g
    torch.cuda.empty_cache()
