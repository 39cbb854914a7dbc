"""GPU replay of tests/golden/*.npz — fixtures produced by the UNMODIFIED
reference (oracle/make_golden.py) — through the device path.

Each fixture holds, for every step, the SHA-256 of the reference's state
(selection indices + values, EF codes, bucket lo/hi, θ) and its StepReport.
The drop-in MicroAdamOptimizer (fp64 θ/g/window on the device, strict
finiteness; blockwise or global Top-K as the fixture was made) must hit the
same digest at every step — parity pinned on the GPU box, where
/root/reference does not exist. Anchors: optim.cpp:164-190 (step),
compress.cpp:39-85 (Top-K), quantize.cpp:7-178 (EF), window.cpp:14-46.
"""
import glob
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _grads(meta, step):
    if meta["generator"] == "zeros":
        return np.zeros(meta["dim"])
    return oracle.synth(42, step, 0, meta["dim"], meta["grad_dtype"], levels=meta["generator"] == "levels")


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))),
                         ids=lambda p: os.path.basename(p)[:-4])
def test_device_replays_golden(path):
    from paper_2405_15593_b200 import MicroAdamOptimizer
    z = np.load(path)
    meta = json.loads(str(z["meta"]))
    d = meta["dim"]
    opt = MicroAdamOptimizer(oracle.synth(1, 0, 0, d, meta["grad_dtype"]), meta["hp"],
                             blockwise=meta["blockwise"])
    for s in range(1, meta["steps"] + 1):
        rep = opt.step(_grads(meta, s))
        sel = opt.last_selection()
        eb = opt.error_buffer()
        got = _digest(np.asarray(sel.indices, np.int64), np.asarray(sel.values, np.float64), eb.codes,
                      np.asarray(eb.lo, np.float64), np.asarray(eb.hi, np.float64),
                      np.asarray(opt.params(), np.float64))
        assert got == str(z["digests"][s - 1]), f"{meta['name']}: state digest differs at step {s}"
        r = z["reports"][s - 1]
        assert rep.update_nnz == int(r[3]), f"update_nnz @ {s}"
        for k, want in zip(("grad_norm", "error_norm", "empirical_q"), r[:3]):
            assert abs(getattr(rep, k) - want) <= 1e-12 * max(abs(want), 1e-300), (k, s)
    assert np.array_equal(np.asarray(opt.params(), np.float64).view(np.uint64),
                          np.asarray(z["params"], np.float64).view(np.uint64))
