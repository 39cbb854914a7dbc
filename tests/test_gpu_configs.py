"""Legal reference configurations outside the lean kernel's shapes.

Buckets that straddle Top-K blocks: QuantizedErrorBuffer::encode buckets the
whole vector (quantize.cpp:142-162) independently of the Top-K blocks
(compress.cpp:73-85), so any B_q >= 1 is legal with any B_d — including the
paper's B_q = 100,000. The device selects per block
(generic kernel, selection marked in a bitmap) and re-quantizes per bucket of
the whole vector (requant_buckets_kernel). fp64: bit-exact against the
UNMODIFIED reference every step; bf16/f32: bit-exact against the composed
oracle; StepReport within 1e-12 (the error norm is summed per bucket).
"""
import pytest

import oracle
from tests.conftest import cuda_available
from tests.test_gpu_parity import run_parity

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


@pytest.mark.parametrize("d,block,bucket", [
    (100_003, 4096, 100),       # B_q ∤ B_d
    (300_007, 4096, 100_000),   # the paper's bucket: one bucket spans ~25 blocks
    (20_011, 1001, 7),          # odd block, odd bucket (buckets share code bytes)
    (50_000, 4096, 4095),
])
def test_straddling_buckets_fp64_vs_unmodified_reference(d, block, bucket):
    hp = dict(lr=1e-2, window=4, block=block, bucket=bucket)
    run_parity(d, hp, gdt="f64", pdt="f64", vdt="f64", steps=8,
               check_reference=oracle.reference_available(), report_every=3)


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_straddling_buckets_low_precision_vs_composed_oracle(dt):
    hp = dict(lr=1e-2, window=5, block=4096, bucket=100)
    run_parity(120_001, hp, gdt=dt, pdt=dt, vdt="bf16", steps=10)


def test_straddling_buckets_host_path():
    """ma_step_host (the drop-in host-buffer call) on a bucket-split handle."""
    import numpy as np
    from paper_2405_15593_b200 import MicroAdamOptimizer
    d, hp = 30_000, dict(lr=1e-2, window=3, block=4096, bucket=1000)
    th0 = oracle.synth(1, 0, 0, d)
    opt = MicroAdamOptimizer(th0, hp, blockwise=True)
    orc = oracle.Oracle(th0, hp)
    for s in range(1, 6):
        g = oracle.synth(42, s, 0, d)
        opt.step(g)
        orc.step(g, hp["lr"])
    assert np.array_equal(opt.params().view(np.uint64), orc.state().params.view(np.uint64))


@pytest.mark.parametrize("d,density,m,steps,dt", [
    (4096 * 4 + 100, 0.002, 300, 320, "bf16"),  # lean kernel (+ generic tail), rows > 255 in the dup lists
    (4096 * 4, 0.01, 600, 610, "f32"),          # staged rows do not fit: the exact warp kernel alone
    (4096 * 4, 0.0005, 1024, 1030, "bf16"),     # the longest window on device
])
def test_long_windows_vs_composed_oracle(d, density, m, steps, dt):
    # HyperParams::validate only needs window >= 1 (optim.cpp:13); the rows are
    # summed in physical slot order (window.cpp:32-39) with weights β^(t - stamp)
    hp = dict(lr=1e-2, window=m, density=density)
    run_parity(d, hp, gdt=dt, pdt=dt, vdt="bf16", steps=steps, check_every=97)


def test_long_window_fp64_vs_unmodified_reference():
    hp = dict(lr=1e-2, window=270, density=0.004)
    run_parity(4096 * 3, hp, gdt="f64", pdt="f64", vdt="f64", steps=280, check_every=70,
               check_reference=oracle.reference_available())


@pytest.mark.parametrize("d,block,bucket,density", [
    (3 * 16384 + 1000, 16384, 64, 0.01),     # B_d > 8192: the big-block kernel
    (2 * 32767 + 5, 32767, 100, 0.005),      # the reference's largest block (compress.hpp:23)
    (20_000, 10_000, 4096, 0.02),
    (9_000, 32767, 64, 0.01),                 # one block of d > 8192 (block = min(B_d, d))
])
def test_big_blocks_fp64_vs_unmodified_reference(d, block, bucket, density):
    hp = dict(lr=1e-2, window=4, block=block, bucket=bucket, density=density)
    run_parity(d, hp, gdt="f64", pdt="f64", vdt="f64", steps=7,
               check_reference=oracle.reference_available(), report_every=3)


def test_big_blocks_bf16_vs_composed_oracle():
    hp = dict(lr=1e-2, window=5, block=20_000, bucket=64, density=0.01)
    run_parity(70_000, hp, gdt="bf16", pdt="bf16", vdt="bf16", steps=9)


def test_big_block_tie_heavy():
    # 16-level gradients: many exact |a| ties at the k_b-th key (lowest indices win)
    hp = dict(lr=1e-2, window=3, block=12_288, bucket=64, density=0.01)
    run_parity(3 * 12_288, hp, gdt="f64", pdt="f64", vdt="f64", steps=5, levels=True,
               check_reference=oracle.reference_available())
