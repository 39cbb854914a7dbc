#!/usr/bin/env python
"""Time the lean kernel's two halves separately (diagnostic, not a bench line):
PH 1 = EF decode / Top-K / window row / re-quantization (ma_step_front over all
blocks), PH 2 = ADAM_STATS + update (ma_step_stats), vs the fused ma_step.
usage: phase_split.py [dim] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_15593_b200 as ma  # noqa: E402

d = int(float(sys.argv[1])) if len(sys.argv) > 1 else 6_738_415_616
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 14
L = ma.lib()
s = torch.cuda.current_stream().cuda_stream
p = torch.empty(d, dtype=torch.bfloat16, device="cuda")
g = torch.empty(d, dtype=torch.bfloat16, device="cuda")
ma._capi.check(L.ma_fill_synthetic(p.data_ptr(), 2, d, 1, 0, 0, 0, s))
res = {}
for mode in ("fused", "split"):
    eng = ma.MicroAdam(d, dict(), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
    nb = d // 4096
    stage = eng.stage_buffers(nb) if mode == "split" else None
    t = []
    for i in range(steps):
        ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), 2, d, 42, i + 1, 0, 0, s))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        if mode == "fused":
            eng.step(p, g, 1e-3)
            ev[1].record()
        else:
            eng.step_front(g, 0, nb, stage)
            ev[1].record()
            eng.step_stats(p, 1e-3)
        ev[2].record()
        torch.cuda.synchronize()
        t.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
    tail = t[10:]
    a = sum(x for x, _ in tail) / len(tail)
    b = sum(y for _, y in tail) / len(tail)
    res[mode] = (a, b)
    print(f"{mode:6s} d={d:,}: first {a:8.3f} ms  second {b:8.3f} ms  (steps 11..{steps}, window full)", flush=True)
    del eng, stage
    torch.cuda.empty_cache()
