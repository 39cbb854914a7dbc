#!/usr/bin/env python
"""Debug: first-step Top-K of the device path vs the oracle, per block (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from tests.test_gpu_parity import _dev, make_engine  # noqa: E402

d = 50_000
rng = np.random.default_rng(5)
spikes = rng.choice(d, 400, replace=False)


def g(s):
    x = oracle.synth(11, s, 0, d) * 1e-3
    x[spikes] += 50.0 + s
    return x


hp = dict(lr=1e-2, window=12)
kernel = sys.argv[1] if len(sys.argv) > 1 else "fast"
theta0 = oracle.synth(1, 0, 0, d, "f32")
orc = oracle.Oracle(theta0, hp, param_dtype="f32", value_dtype="bf16")
eng = make_engine(kernel, d, hp, param_dtype="f32", grad_dtype="bf16", value_dtype="bf16")
params = _dev(theta0, "f32")
for s in range(1, 4):
    gg = g(s)
    gd = _dev(gg, "bf16")
    gb = gd.double().cpu().numpy()
    eng.step(params, gd, 1e-2)
    orc.step(gg, 1e-2)
    torch.cuda.synchronize()
    so = orc.state()
    win = eng.window()
    step, head, filled, stamps = eng.counters()
    slot = (head + orc.m - 1) % orc.m
    mine, want = win.indices[slot], so.last_idx
    if np.array_equal(mine, want):
        print("step", s, "ok")
        continue
    bad = np.nonzero(mine != want)[0]
    print("step", s, "mismatch at", bad[:10], "n", len(bad))
    b = want[bad[0]] // 4096
    sel_m = mine[(mine // 4096) == b]
    sel_w = want[(want // 4096) == b]
    print("block", b, "mine", len(sel_m), "want", len(sel_w))
    print(" only mine:", sorted(set(sel_m) - set(sel_w)), [gb[i] for i in sorted(set(sel_m) - set(sel_w))])
    print(" only want:", sorted(set(sel_w) - set(sel_m)), [gb[i] for i in sorted(set(sel_w) - set(sel_m))])
    blk = np.abs(gb[b * 4096:(b + 1) * 4096])
    order = np.argsort(-blk, kind="stable")
    print(" top 45 |g|:", [(int(b * 4096 + i), blk[i]) for i in order[:45]])
    print(" mine order ok:", np.all(np.diff(sel_m) > 0))
    break
