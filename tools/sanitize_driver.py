#!/usr/bin/env python
"""Small runs of every kernel family for compute-sanitizer (tools/r2_sanitize.sh):
lean (default), exact warp (MA_WARP_EXACT=1 in the env), generic (3-bit EF),
global Top-K (blockwise=False), sparse-propagation phases, fused reduce-scatter."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_15593_b200 as ma  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "lean"
d = 4096 * 64 + 1000
L = ma.lib()
s = torch.cuda.current_stream().cuda_stream


def fill(t, seed, step):
    ma._capi.check(L.ma_fill_synthetic(t.data_ptr(), 2, t.numel(), seed, step, 0, 0, s))


hp = dict(window=4)
if which == "generic":
    hp["bits"] = 3
eng = ma.MicroAdam(d, hp, param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16",
                   blockwise=(which != "global"))
p = torch.empty(d, dtype=torch.bfloat16, device="cuda")
g = torch.empty(d, dtype=torch.bfloat16, device="cuda")
fill(p, 1, 0)
for i in range(6):
    fill(g, 42, i + 1)
    if which == "sparse":
        nb = d // 4096
        eng2 = eng
        st = eng.stage_buffers(nb)
        dd = nb * 4096
        e = ma.MicroAdam(dd, hp, param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
        pp = p[:dd].clone()
        e.step_front(g[:dd], 0, nb, st)
        e.step_stats(pp, 1e-3)
    elif which == "reduce":
        g2 = g.clone()
        eng.step_reduce(p, g, [g, g2], 0.5, 1e-3)
    else:
        eng.step(p, g, 1e-3)
eng.synchronize()
torch.cuda.synchronize()
print("ok", which, eng.kernel_launches())
