"""ma_step_host (the reference-facing host-buffer step) against ma_step on the
device, bit for bit.

The chunked host path streams g up and θ back; with MA_HOST_SPARSE=1 it
returns only the window ring indices plus the θ values gathered at them,
scattered into the caller's buffer on host threads (θ changes only at window
coordinates, optim.cpp:183-187). Checked: several 64 MB chunks with a tail
block, ring wrap-around (steps > m), bf16 / f32 / f64 θ, the default dense
return, and a switch to a fresh host buffer mid-run (dense fallback: the
sparse return is only valid into the buffer that already holds the device θ).
"""
import os

import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

BLK = 4096


def _tdt(dt):
    import torch
    return {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[dt]


def _pair(d, hp, dt):
    from paper_2405_15593_b200 import MicroAdam
    return (MicroAdam(d, hp, param_dtype=dt, grad_dtype=dt, value_dtype="bf16"),
            MicroAdam(d, hp, param_dtype=dt, grad_dtype=dt, value_dtype="bf16"))


def _run(d, hp, dt, steps, dense=False, swap_at=None):
    """Sparse return (MA_HOST_SPARSE=1) unless dense."""
    import torch
    gen = torch.Generator(device="cuda").manual_seed(11)
    theta = torch.randn(d, generator=gen, device="cuda").to(_tdt(dt))
    dev, host = _pair(d, hp, dt)
    p_dev = theta.clone()
    h_p = theta.cpu().pin_memory()
    h_g = torch.empty(d, dtype=_tdt(dt)).pin_memory()
    if not dense:
        os.environ["MA_HOST_SPARSE"] = "1"
    try:
        for s in range(steps):
            g = (torch.randn(d, generator=gen, device="cuda") * (1 + s)).to(_tdt(dt))
            h_g.copy_(g.cpu())
            dev.step(p_dev, g, hp["lr"])
            if swap_at == s:  # a different host buffer (contents ignored: the device θ is authoritative)
                h_p = torch.zeros_like(h_p).pin_memory()
            host.step_host(h_p, h_g, hp["lr"])
            torch.cuda.synchronize()
            iv = {"bf16": torch.int16, "f32": torch.int32, "f64": torch.int64}[dt]
            assert torch.equal(h_p.view(iv), p_dev.cpu().view(iv)), f"θ differs after step {s + 1}"
    finally:
        os.environ.pop("MA_HOST_SPARSE", None)
    assert np.array_equal(dev.error_buffer().codes, host.error_buffer().codes)
    assert np.array_equal(dev.window().indices, host.window().indices)


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_step_host_sparse_return_matches_device_multichunk(dt):
    # bf16: 8192 blocks per 64 MB chunk; 2.5 chunks + a ragged tail block
    nblk = 20480 if dt == "bf16" else 10240
    d = nblk * BLK + 1234
    _run(d, dict(lr=1e-3, window=3), dt, steps=5)


def test_step_host_f64_and_wide_window():
    _run(300 * BLK + 77, dict(lr=1e-2, window=10, density=0.02), "f64", steps=12)


def test_step_host_dense_return_default():
    _run(9000 * BLK, dict(lr=1e-3, window=4), "bf16", steps=6, dense=True)


def test_step_host_new_buffer_falls_back_to_dense():
    _run(700 * BLK + 5, dict(lr=1e-3, window=3), "bf16", steps=6, swap_at=3)
