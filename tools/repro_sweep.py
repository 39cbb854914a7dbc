"""Small repro of the 13B sweep points (heavy-tailed stream) vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_2405_15593_b200 as ma

def run(nblk, tail, density, window, steps, mode):
    dim = nblk * 4096 + tail
    hp = dict(lr=1e-3, density=density, window=window)
    eng = ma.MicroAdam(dim, hp, param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
    orc = oracle.Oracle(oracle.synth(1, 0, 0, dim, "bf16"), hp, param_dtype="bf16", value_dtype="bf16")
    p = torch.from_numpy(oracle.synth(1, 0, 0, dim, "bf16")).to(torch.bfloat16).cuda()
    for s in range(1, steps + 1):
        g = oracle.synth(42, s, 0, dim, "bf16", heavy=mode == 2)
        eng.step(p, torch.from_numpy(g).to(torch.bfloat16).cuda(), 1e-3)
        orc.step(g, 1e-3)
        torch.cuda.synchronize()
        so = orc.state()
        got = p.double().cpu().numpy()
        ok = np.array_equal(got.view(np.uint64), so.params.view(np.uint64))
        eb = eng.error_buffer()
        okc = np.array_equal(eb.codes, so.codes)
        if not (ok and okc):
            print("MISMATCH", dim, density, window, "step", s, ok, okc, flush=True)
            return False
    print("ok", dim, density, window, mode, flush=True)
    return True

for args in [(40, 1024, 0.05, 20, 24, 2), (40, 0, 0.05, 20, 24, 2), (40, 1024, 0.05, 20, 24, 0),
             (40, 1024, 0.001, 5, 9, 2), (40, 1024, 0.02, 10, 14, 2)]:
    run(*args)
