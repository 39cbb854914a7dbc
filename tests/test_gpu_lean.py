"""Parity of the fp32-screened ("lean") warp kernel.

The lean kernel (ma_warp.cu: microadam_step_lean) runs for bf16 / f32
gradients without a StepReport. It decodes the EF and re-quantizes in fp32
with proven error bounds and re-decides in fp64 whatever fp32 cannot settle,
so its results must be bit-identical to the reference algorithm. These tests
target the inputs where the bounds are tight or void: scale jumps (threshold
drift), spikes (wide buckets), magnitudes at the fp32 range limits
(subnormals, overflow of a32), coarse value grids (exact ties in min / max
and in the 4-bit quotient), and a direct comparison against the exact warp
kernel at a size the oracle would be slow for.
"""
import numpy as np
import pytest

import oracle
from tests.conftest import cuda_available
from tests.test_gpu_parity import _bits, _dev, _host, _torch, make_engine, run_parity

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

D = 4096 * 7 + 4096 // 2  # whole blocks + a generic-kernel tail


def test_scale_jumps_f32():
    scales = [1.0, 2.0 ** 20, 2.0 ** 20, 2.0 ** -20, 1.0, 1.0, 3.0, 1.0, 2.0 ** -3, 1.0]
    run_parity(D, dict(lr=1e-2), gdt="f32", pdt="f32", vdt="bf16", steps=len(scales),
               grad_fn=lambda s: oracle.synth(9, s, 0, D) * scales[s - 1])


def test_spiky_f32():
    rng = np.random.default_rng(3)

    def g(s):
        x = oracle.synth(13, s, 0, D) * 1e-4
        idx = rng.choice(D, 300, replace=False)
        x[idx] = np.round(rng.standard_normal(300) * 1e3) / 8
        return x
    run_parity(D, dict(lr=1e-2), gdt="f32", pdt="f32", vdt="bf16", steps=10, grad_fn=g)


@pytest.mark.parametrize("scale", [2.0 ** -140, 2.0 ** -120, 2.0 ** -100, 2.0 ** 100, 2.0 ** 126])
def test_fp32_range_limits(scale):
    # f32 subnormal gradients, values near FLT_MAX (a = g + e overflows fp32)
    run_parity(D, dict(lr=1e-3), gdt="f32", pdt="f32", vdt="f32", steps=6,
               grad_fn=lambda s: oracle.synth(7, s, 0, D) * scale)


@pytest.mark.parametrize("grid", [0.25, 2.0 ** -12])
def test_coarse_value_grid_ties(grid):
    # values on a coarse grid: exact ties in |a|, in bucket min / max and
    # quotients landing exactly on half-integers
    run_parity(D, dict(lr=1e-2), gdt="f32", pdt="f32", vdt="bf16", steps=10,
               grad_fn=lambda s: np.round(oracle.synth(21, s, 0, D) / grid) * grid)


def test_bf16_constant_blocks_and_two_level_buckets():
    def g(s):
        x = np.zeros(D)
        x[: 4096] = 1.5                                   # constant block
        x[4096: 8192] = np.where(np.arange(4096) % 2, 2.0, -2.0)  # two-valued buckets
        x[8192:] = oracle.synth(4, s, 0, D - 8192)
        return x
    run_parity(D, dict(lr=1e-2), gdt="bf16", pdt="bf16", vdt="bf16", steps=8, grad_fn=g)


def test_bucket32_f32():
    run_parity(D, dict(lr=1e-2, bucket=32), gdt="f32", pdt="f32", vdt="bf16", steps=10)


def test_long_run_bf16():
    run_parity(4096 * 4, dict(lr=1e-3), gdt="bf16", pdt="bf16", vdt="bf16", steps=30)


def test_lean_matches_exact_warp_kernel_at_scale():
    """Lean vs exact warp kernel, every state array bit-for-bit, 8M params."""
    torch = _torch()
    d = 4096 * 2048
    hp = dict(lr=1e-3)
    engs = {k: make_engine(k, d, hp, param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
            for k in ("fast", "warp_exact")}
    theta0 = oracle.synth(1, 0, 0, d, "bf16")
    params = {k: _dev(theta0, "bf16") for k in engs}
    for s in range(1, 15):
        g = _dev(oracle.synth(42, (s - 1) % 6 + 1, 0, d, "bf16"), "bf16")  # repeats -> duplicates
        for k, e in engs.items():
            e.step(params[k], g, 1e-3)
        torch.cuda.synchronize()
        assert torch.equal(params["fast"], params["warp_exact"]), f"θ @ {s}"
    a, b = engs["fast"], engs["warp_exact"]
    assert np.array_equal(a.error_buffer().codes, b.error_buffer().codes)
    assert np.array_equal(_bits(a.error_buffer().lo), _bits(b.error_buffer().lo))
    assert np.array_equal(_bits(a.error_buffer().hi), _bits(b.error_buffer().hi))
    wa, wb = a.window(), b.window()
    assert np.array_equal(wa.indices, wb.indices)
    assert np.array_equal(_bits(wa.values), _bits(wb.values))
    assert np.array_equal(_bits(_host(params["fast"])), _bits(_host(params["warp_exact"])))


@pytest.mark.parametrize("lr,tscale", [(1e-3, 1.0), (0.5, 1.0), (1e-2, 2.0 ** -12), (1e-3, 0.0),
                                       (1e-3, 2.0 ** -110), (1e-1, 2.0 ** 100)])
def test_bf16_theta_update_screen(lr, tscale):
    # the fp32 θ-update screen (|lr u| vs |θ|, rounding midpoints, θ = 0,
    # exponents outside the screened range) must reproduce the fp64 update
    d = 4096 * 4
    th = oracle.synth(1, 0, 0, d) * tscale
    run_parity(d, dict(lr=lr), gdt="bf16", pdt="bf16", vdt="bf16", steps=12, theta0=th)


def test_bf16_theta_f32_window_values():
    run_parity(4096 * 4, dict(lr=1e-2), gdt="bf16", pdt="bf16", vdt="f32", steps=12)


@pytest.mark.parametrize("per_block,pdt", [(5, "bf16"), (5, "f32"), (20, "bf16"), (60, "bf16")])
def test_duplicate_coordinates_chunked(per_block, pdt):
    # a few coordinates per block win every step: 32 < duplicate entries <= 256
    # with <= 64 coordinates (chunked match.any path), and beyond (fallback)
    d = 4096 * 6
    rng = np.random.default_rng(per_block)
    spikes = np.concatenate([b * 4096 + rng.choice(4096, per_block, replace=False) for b in range(6)])

    def g(s):
        x = oracle.synth(17, s, 0, d)
        x[spikes] += 40.0 + s
        return x
    run_parity(d, dict(lr=1e-2, window=12), gdt="bf16", pdt=pdt, vdt="bf16", steps=16, grad_fn=g)


@pytest.mark.parametrize("density,dt", [(0.02, "bf16"), (0.03, "f32"), (0.03125, "bf16"), (0.05, "bf16"),
                                        (0.0625, "f32")])
def test_wide_kb_lean_variant(density, dt):
    # k_b in (64, 128] (densities 1.6%-3.1%): the 8-slot lean variant (k_b = 128
    # at 3.125%); k_b in (128, 256] (to 6.25%): the 16-slot one
    run_parity(4096 * 6 + 900, dict(lr=1e-2, density=density, window=6), gdt=dt, pdt=dt, vdt="bf16",
               steps=10)


@pytest.mark.parametrize("density", [0.025, 0.04])
def test_wide_kb_tie_heavy(density):
    run_parity(4096 * 4, dict(lr=1e-2, density=density, window=4), gdt="f32", pdt="f32", vdt="bf16",
               steps=8, levels=True)
