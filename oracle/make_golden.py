#!/usr/bin/env python
"""Generate tests/golden/*.npz by running the UNMODIFIED reference
(oracle/_ref/libmicroadam_ref.so, compiled from /root/reference/proj/src) on
the include/ma_synth.h input stream. TEST INFRASTRUCTURE ONLY.

Each fixture stores the config, per-step SHA-256 digests of the reference's
state after every step (selection indices+values, EF codes, bucket lo/hi, θ)
and the final state arrays. tests/test_oracle.py replays the same inputs
through the C restatement and (on a GPU box) tests/test_gpu_golden.py through
the CUDA path, so parity stays pinned where /root/reference does not exist.

    python oracle/make_golden.py     # needs /root/reference (this container)
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

# name -> (dim, hp, blockwise, grad dtype, steps, generator)
CASES = {
    "default_10k": (10_000, dict(lr=1e-3), True, "f32", 20, "normal"),
    "tail_4099_b512_q16_m3": (4099, dict(block=512, bucket=16, window=3, lr=1e-2), True, "f32", 15,
                              "normal"),
    "odd_37_b8_q4": (37, dict(block=8, bucket=4, window=2, density=0.25, lr=1e-2), True, "f64", 8,
                     "normal"),
    "ties_5000_levels": (5000, dict(block=1024, window=4, lr=1e-2), True, "f32", 10, "levels"),
    "zeros_3000": (3000, dict(window=3, lr=1e-2), True, "f32", 5, "zeros"),
    "global_2000_k20": (2000, dict(k=20, window=5, lr=1e-2), False, "f64", 8, "normal"),
    "bf16_grads_20000_m5_d5pct": (20_000, dict(window=5, density=0.05, lr=1e-3), True, "bf16", 12,
                                  "normal"),
}


def grads(kind, dim, step, dtype):
    if kind == "zeros":
        return np.zeros(dim)
    return oracle.synth(42, step, 0, dim, dtype, levels=(kind == "levels"))


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def state_digest(st):
    return digest(st.last_idx, st.last_val, st.codes, st.lo, st.hi, st.params)


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, (dim, hp, blockwise, gdt, steps, kind) in CASES.items():
        theta0 = oracle.synth(1, 0, 0, dim, gdt)
        ref = oracle.Reference(theta0, hp, blockwise=blockwise)
        digests, reports = [], []
        for s in range(1, steps + 1):
            rep = ref.step(grads(kind, dim, s, gdt))
            st = ref.state()
            digests.append(state_digest(st))
            reports.append([rep["grad_norm"], rep["error_norm"], rep["empirical_q"],
                            rep["update_nnz"]])
        st = ref.state()
        meta = dict(name=name, dim=dim, hp=hp, blockwise=blockwise, grad_dtype=gdt, steps=steps,
                    generator=kind, theta0="synth(seed=1, step=0)",
                    grads="synth(seed=42, step=s) rounded to grad_dtype",
                    source="unmodified reference (oracle/_ref) via oracle/make_golden.py")
        np.savez_compressed(
            os.path.join(OUT, f"{name}.npz"), meta=json.dumps(meta), digests=np.array(digests),
            reports=np.array(reports), params=st.params, codes=st.codes, lo=st.lo, hi=st.hi,
            step=st.step, head=st.head, filled=st.filled, stamps=st.stamps, win_idx=st.win_idx,
            win_val=st.win_val, last_idx=st.last_idx, last_val=st.last_val)
        print(f"{name}: {steps} steps, final digest {digests[-1][:16]}")


if __name__ == "__main__":
    main()
