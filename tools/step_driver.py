#!/usr/bin/env python
"""Minimal driver for profiling: N MicroAdam steps on one GPU.

    python tools/step_driver.py --dim 110000000 --dtype bf16 --steps 3
Used under ncu (tools/r2_ncu_kern.sh, tools/r2_evidence.sh); never a bench number.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2405_15593_b200 as ma  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=110_000_000)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--vdtype", default="bf16")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--density", type=float, default=0.01)
ap.add_argument("--window", type=int, default=10)
ap.add_argument("--levels", action="store_true")
a = ap.parse_args()
tdt = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[a.dtype]
code = {"f64": 0, "f32": 1, "bf16": 2}[a.dtype]
eng = ma.MicroAdam(a.dim, dict(density=a.density, window=a.window), param_dtype=a.dtype,
                   grad_dtype=a.dtype, value_dtype=a.vdtype)
p = torch.empty(a.dim, dtype=tdt, device="cuda")
g = torch.empty(a.dim, dtype=tdt, device="cuda")
L = ma.lib()
s = torch.cuda.current_stream().cuda_stream
ma._capi.check(L.ma_fill_synthetic(p.data_ptr(), code, a.dim, 1, 0, 0, 0, s))
for i in range(a.steps):
    ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), code, a.dim, 42, i + 1, 0, int(a.levels), s))
    eng.step(p, g, 1e-3)
eng.synchronize()
print("ok", eng.kernel_launches())
