"""Quick oracle check of the default step kernel on small configs (debug aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2405_15593_b200 as ma

TDT = {"bf16": torch.bfloat16, "f32": torch.float32}


def run(nblk, tail, hp, dt, steps, mode, vdt="bf16"):
    dim = nblk * 4096 + tail
    eng = ma.MicroAdam(dim, hp, param_dtype=dt, grad_dtype=dt, value_dtype=vdt)
    th0 = oracle.synth(1, 0, 0, dim, dt)
    orc = oracle.Oracle(th0, hp, param_dtype=dt, value_dtype=vdt)
    p = torch.from_numpy(th0).to(TDT[dt]).cuda()
    lr = hp.get("lr", 1e-3)
    for s in range(1, steps + 1):
        g = oracle.synth(42, s, 0, dim, dt, heavy=mode == 2, levels=mode == 1)
        eng.step(p, torch.from_numpy(g).to(TDT[dt]).cuda(), lr)
        orc.step(g, lr)
        torch.cuda.synchronize()
        so = orc.state()
        eb = eng.error_buffer()
        win = eng.window()
        msgs = []
        head = eng.counters()[1]
        slot = (head + orc.m - 1) % orc.m
        if not np.array_equal(win.indices[slot], so.last_idx):
            bad = np.flatnonzero(win.indices[slot] != so.last_idx)
            msgs.append(f"topk idx @pos {bad[:5]} got {win.indices[slot][bad[:5]]} want {so.last_idx[bad[:5]]}")
        if not np.array_equal(eb.codes, so.codes):
            bad = np.flatnonzero(eb.codes != so.codes)
            msgs.append(f"codes @byte {bad[:5]} got {eb.codes[bad[:5]]} want {so.codes[bad[:5]]} (n={bad.size})")
        if not np.array_equal(eb.lo.view(np.uint64), so.lo.view(np.uint64)):
            bad = np.flatnonzero(eb.lo.view(np.uint64) != so.lo.view(np.uint64))
            msgs.append(f"lo @bucket {bad[:5]} got {eb.lo[bad[:3]]} want {so.lo[bad[:3]]} (n={bad.size})")
        if not np.array_equal(eb.hi.view(np.uint64), so.hi.view(np.uint64)):
            bad = np.flatnonzero(eb.hi.view(np.uint64) != so.hi.view(np.uint64))
            msgs.append(f"hi @bucket {bad[:5]} got {eb.hi[bad[:3]]} want {so.hi[bad[:3]]} (n={bad.size})")
        for r in range(so.filled):
            if not np.array_equal(win.indices[r], so.win_idx[r]) or not np.array_equal(
                    win.values[r].view(np.uint64), so.win_val[r].view(np.uint64)):
                msgs.append(f"window row {r}")
                break
        got = p.double().cpu().numpy()
        bad = np.flatnonzero(got.view(np.uint64) != so.params.view(np.uint64))
        if bad.size:
            msgs.append(f"theta @ {bad[:5]} got {got[bad[:3]]} want {so.params[bad[:3]]} (n={bad.size})")
        if msgs:
            print(f"MISMATCH dim={dim} hp={hp} dt={dt} mode={mode} step {s}: " + "; ".join(msgs), flush=True)
            return False
    print(f"ok dim={dim} hp={hp} dt={dt} mode={mode} steps={steps} dbg={eng.debug_counters() if os.environ.get('MA_DEBUG_COUNTERS') else ''}", flush=True)
    return True


if __name__ == "__main__":
    oracle.build()
    cases = [
        (8, 0, dict(lr=1e-3, window=4), "bf16", 6, 0),
        (40, 1000, dict(lr=1e-3), "bf16", 14, 0),
        (40, 1000, dict(lr=1e-3), "bf16", 14, 2),
        (40, 0, dict(lr=1e-2, window=3), "f32", 8, 0),
        (40, 0, dict(lr=1e-2, window=3), "f32", 8, 2),
        (20, 0, dict(lr=1e-2, window=5), "bf16", 8, 1),
        (40, 1024, dict(lr=1e-3, density=0.05, window=20), "bf16", 24, 2),
        (40, 1024, dict(lr=1e-3, density=0.001, window=5), "bf16", 9, 2),
        (40, 1024, dict(lr=1e-3, density=0.02, window=10), "bf16", 14, 2),
    ]
    only = sys.argv[1:]
    for i, c in enumerate(cases):
        if only and str(i) not in only:
            continue
        t = time.time()
        run(*c)
