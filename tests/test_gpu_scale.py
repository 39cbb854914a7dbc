"""Parity at the BASELINE configurations themselves, on sampled block ranges.

The blockwise step is block-independent (compress.cpp:73-85: each block's
Top-K, its buckets' re-quantization and its window columns depend only on
that block's g and EF), and the host counters / weights are global
(window.cpp:28-46). So the composed oracle run on just the sampled blocks —
fed the same counter-based gradient slices (include/ma_synth.h) — must equal
the device's full-size run on those blocks, bit for bit: EF codes, (lo, hi),
every window row (indices and values) and θ.

Sampled ranges cover the first blocks, ranges straddling element offsets
2^31 and 2^32 (64-bit indexing), the middle and the last block. The gradient
stream is the bench's own (bench.grad_source: step i reads ma_synth step
(i % 8) + 1 at a shifted offset), Gaussian-like or heavy-tailed with
per-block scales (ma_synth_heavy). Anchors: optim.cpp:164-190,
compress.cpp:73-85, quantize.cpp:142-162, window.cpp:28-46.
"""
import numpy as np
import pytest

import oracle
from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

MA_DT = {"f64": 0, "f32": 1, "bf16": 2}
B = 8  # resident gradient buffers of the bench stream


def _bits(x):
    return np.asarray(x, np.float64).view(np.uint64)


def _ranges(nblocks, block, per=4):
    """Sampled block ranges: first, around element 2^31 and 2^32, middle, last."""
    want = [0]
    for e in (1 << 31, 1 << 32):
        b = e // block
        if b + per // 2 < nblocks:
            want.append(max(0, b - per // 2))
    want += [nblocks // 2, nblocks - per]
    out = []
    for b0 in sorted(set(want)):
        b0 = max(0, min(b0, nblocks - per))
        if out and b0 < out[-1][1]:
            continue
        out.append((b0, min(nblocks, b0 + per)))
    return out


def run_sampled(dim, hp, *, dt, vdt="bf16", steps=25, mode=0, per=4, check_every=8):
    import torch

    import bench
    import paper_2405_15593_b200 as ma

    oracle.build()
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[dt]
    eng = ma.MicroAdam(dim, hp, param_dtype=dt, grad_dtype=dt, value_dtype=vdt)
    lay = eng.layout
    lib = ma.lib()
    params = torch.empty(dim, dtype=tdt, device="cuda")
    grads = torch.empty(dim, dtype=tdt, device="cuda")

    def fill(t, seed, step, offset, fmode):
        ma._capi.check(lib.ma_fill_synthetic(t.data_ptr(), MA_DT[dt], t.numel(), seed, step, offset, fmode,
                                             None))

    fill(params, 1, 0, 0, 0)
    ranges = _ranges(lay.num_blocks, lay.block, per)
    blk = lay.block
    orcs = []
    for b0, b1 in ranges:
        e0, e1 = b0 * blk, min(dim, b1 * blk)
        th0 = oracle.synth(1, 0, e0, e1 - e0, dt)
        orcs.append(oracle.Oracle(th0, hp, param_dtype=dt, value_dtype=vdt))
    lr = hp.get("lr", 1e-3)
    for s in range(1, steps + 1):
        j, off = bench.grad_source(s - 1, B)
        fill(grads, 42, j, off, mode)
        eng.step(params, grads, lr)
        for (b0, b1), orc in zip(ranges, orcs):
            e0, e1 = b0 * blk, min(dim, b1 * blk)
            orc.step(oracle.synth(42, j, off + e0, e1 - e0, dt, heavy=mode == 2, levels=mode == 1), lr)
        if s % check_every and s != steps:
            continue
        torch.cuda.synchronize()
        eng.synchronize()
        step, head, filled, stamps = eng.counters()
        for (b0, b1), orc in zip(ranges, orcs):
            so = orc.state()
            tag = f"{dim:,} blocks [{b0}, {b1}) step {s}"
            assert (step, head, filled) == (so.step, so.head, so.filled), tag
            codes, lo, hi = eng.error_buffer_blocks(b0, b1)
            assert np.array_equal(codes, so.codes), f"EF codes differ: {tag}"
            assert np.array_equal(_bits(lo), _bits(so.lo)), f"EF lo differ: {tag}"
            assert np.array_equal(_bits(hi), _bits(so.hi)), f"EF hi differ: {tag}"
            e0, e1 = b0 * blk, min(dim, b1 * blk)
            for r in range(filled):
                idx, val = eng.window_blocks(r, b0, b1)
                assert np.array_equal(idx, so.win_idx[r] + e0), f"window row {r} indices differ: {tag}"
                assert np.array_equal(_bits(val), _bits(so.win_val[r])), f"window row {r} values differ: {tag}"
            got = params[e0:e1].to(torch.float64).cpu().numpy()
            bad = np.flatnonzero(_bits(got) != _bits(so.params))
            assert bad.size == 0, f"θ differs: {tag} at {bad[:8] + e0}"
    del params, grads
    eng.close()
    torch.cuda.empty_cache()
    return ranges


LLAMA7B = 6_738_415_616
LLAMA13B = 13_015_864_320


def test_headline_7b_bf16_bench_stream():
    """BASELINE configs[3] (the bench's workload): 7B bf16 θ/g/window, 1%, m=10,
    4-bit EF, 25 steps of the bench's gradient stream."""
    ranges = run_sampled(LLAMA7B, dict(lr=1e-3), dt="bf16", steps=25)
    assert any(b0 * 4096 < (1 << 32) <= b1 * 4096 for b0, b1 in ranges)
    assert ranges[-1][1] == LLAMA7B // 4096


def test_headline_7b_bf16_heavy_tailed():
    """Same config, heavy-tailed per-block-scaled gradients (scales 2^-16..2^16
    drifting every 4 steps, 1/64 outliers up to 2^12x)."""
    run_sampled(LLAMA7B, dict(lr=1e-3), dt="bf16", steps=25, mode=2)


def test_bert_110m_f32():
    """BASELINE configs[1]: 110M f32 (tail block of 1,920)."""
    run_sampled(110_000_000, dict(lr=1e-3), dt="f32", steps=14, mode=2)


def test_opt_1_3b_bf16():
    """BASELINE configs[2]: 1.3B bf16 (tail block of 3,328)."""
    run_sampled(1_300_000_000, dict(lr=1e-3), dt="bf16", steps=14)


@pytest.mark.parametrize("density,window", [(0.05, 20), (0.001, 5), (0.02, 10)])
def test_13b_sweep_points(density, window):
    """BASELINE configs[4] sweep points (13B bf16): 5%/m=20 (k_b = 205, the
    wide candidate path), 0.1%/m=5, 2%/m=10."""
    run_sampled(LLAMA13B, dict(lr=1e-3, density=density, window=window), dt="bf16",
                steps=window + 4, mode=2, per=2, check_every=window)
