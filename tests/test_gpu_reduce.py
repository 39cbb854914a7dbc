"""Gradient reduce-scatter fused into the step (ma_step_reduce, SURVEY.md
§8(f) rank 2) on one GPU, with the ranks' gradients as local buffers.

The contract: the step uses g = rn(((s_0 + s_1) + ...) * scale) with fp32
sums for bf16/f32 gradients, writes it into the grads buffer, and is then
bit-identical to ma_step on that g. Checked against a torch restatement of the
reduction followed by the ordinary step: θ, EF codes, window rows and the
written gradient, for 1-8 sources, a ragged tail block, the output aliasing a
source, the unfused fallback (MA_RS_UNFUSED=1, B_q = 32, reports) and bad
arguments.
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


def _reduce(srcs, scale):
    """The reduction ma_step_reduce defines (torch restatement, rank order)."""
    import torch
    wide = torch.float64 if srcs[0].dtype == torch.float64 else torch.float32
    acc = srcs[0].to(wide)
    for s in srcs[1:]:
        acc = acc + s.to(wide)
    acc = acc * torch.tensor(scale, dtype=torch.float32, device=acc.device).to(wide)
    return acc.to(srcs[0].dtype)


def _engines(d, hp, dt, bucket=64):
    from paper_2405_15593_b200 import MicroAdam
    hp = dict(hp, bucket=bucket)
    return (MicroAdam(d, hp, param_dtype=dt, grad_dtype=dt, value_dtype=dt),
            MicroAdam(d, hp, param_dtype=dt, grad_dtype=dt, value_dtype=dt))


def _run(d, hp, dt, nsrc, scale, steps=6, alias=False, bucket=64, unfused=False, report=False):
    import torch
    gen = torch.Generator(device="cuda").manual_seed(5 + nsrc)
    th0 = torch.randn(d, generator=gen, device="cuda").to(_tdt(dt))
    ref, eng = _engines(d, hp, dt, bucket)
    p_ref, p_eng = th0.clone(), th0.clone()
    if unfused:
        os.environ["MA_RS_UNFUSED"] = "1"
    try:
        for s in range(steps):
            srcs = [(torch.randn(d, generator=gen, device="cuda") * (0.5 + r)).to(_tdt(dt)) for r in range(nsrc)]
            g_ref = _reduce(srcs, scale)
            out = srcs[0] if alias else torch.empty_like(srcs[0])
            rr = ref.step(p_ref, g_ref, hp["lr"], report=report)
            re = eng.step_reduce(p_eng, out, srcs, scale, hp["lr"], report=report)
            torch.cuda.synchronize()
            iv = {"bf16": torch.int16, "f32": torch.int32, "f64": torch.int64}[dt]
            assert torch.equal(out.view(iv), g_ref.view(iv)), f"reduced gradient differs at step {s + 1}"
            assert torch.equal(p_eng.view(iv), p_ref.view(iv)), f"θ differs at step {s + 1}"
            if report:
                assert re.update_nnz == rr.update_nnz and re.grad_norm == rr.grad_norm
    finally:
        os.environ.pop("MA_RS_UNFUSED", None)
    assert np.array_equal(eng.error_buffer().codes, ref.error_buffer().codes)
    assert np.array_equal(eng.window().indices, ref.window().indices)


@pytest.mark.parametrize("nsrc", [1, 2, 3, 8])
def test_fused_reduce_bf16_matches_reduce_then_step(nsrc):
    _run(64 * BLK + 1000, dict(lr=1e-3, window=4), "bf16", nsrc, 1.0 / nsrc)


def test_fused_reduce_f32_and_alias():
    _run(40 * BLK, dict(lr=1e-3, window=3), "f32", 5, 0.2, alias=True)


def test_fused_reduce_unit_scale_full_window():
    _run(24 * BLK + 7, dict(lr=1e-2, window=10), "bf16", 4, 1.0, steps=13)


@pytest.mark.parametrize("kw", [dict(unfused=True), dict(bucket=32), dict(report=True)])
def test_unfused_paths_match(kw):
    _run(20 * BLK + 300, dict(lr=1e-3, window=3), "bf16", 3, 1.0 / 3, **kw)


def test_unfused_f64():
    _run(10 * BLK + 9, dict(lr=1e-2, window=3), "f64", 2, 0.5)


def test_bad_source_counts_rejected():
    import torch
    from paper_2405_15593_b200 import MicroAdam
    d = 4 * BLK
    eng = MicroAdam(d, dict(lr=1e-3), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
    p = torch.zeros(d, dtype=torch.bfloat16, device="cuda")
    g = torch.zeros_like(p)
    with pytest.raises(ValueError):
        eng.step_reduce(p, g, [])
    with pytest.raises(ValueError):
        eng.step_reduce(p, g, [g] * 9)
    with pytest.raises(Exception):
        eng.step_reduce(p, g, [g, torch.zeros(d, dtype=torch.float32, device="cuda")])


def test_fused_reduce_on_block_shards():
    # each shard handle reads its element range of every rank's full gradient
    # (sources offset by the shard start, as the symmetric-memory loop does)
    import torch
    from paper_2405_15593_b200 import MicroAdam, sharding
    d, hp, nsrc = 30 * BLK + 123, dict(lr=1e-3, window=3), 4
    gen = torch.Generator(device="cuda").manual_seed(3)
    th0 = torch.randn(d, generator=gen, device="cuda").to(torch.bfloat16)
    full = MicroAdam(d, hp, param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
    p_full = th0.clone()
    shards = []
    for r in range(3):
        b0, b1, e0, e1 = sharding.partition_blocks(d, BLK, 3, r)
        eng = MicroAdam(d, hp, param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16", block_range=(b0, b1))
        shards.append((eng, e0, e1, th0[e0:e1].clone()))
    for s in range(5):
        srcs = [torch.randn(d, generator=gen, device="cuda").to(torch.bfloat16) for _ in range(nsrc)]
        g = _reduce(srcs, 0.25)
        full.step(p_full, g, hp["lr"])
        for eng, e0, e1, p in shards:
            out = torch.empty(e1 - e0, dtype=torch.bfloat16, device="cuda")
            eng.step_reduce(p, out, [x[e0:e1] for x in srcs], 0.25, hp["lr"])
        torch.cuda.synchronize()
        for eng, e0, e1, p in shards:
            assert torch.equal(p.view(torch.int16), p_full[e0:e1].view(torch.int16)), f"shard θ @ {s}"


@pytest.mark.parametrize("dt,nsrc", [("bf16", 4), ("f32", 3)])
def test_fused_reduce_matches_oracle(dt, nsrc):
    """ma_step_reduce against the composed oracle fed the torch-reduced gradient
    (optim.cpp:166-168: the step's a = g + e with g the reduced gradient)."""
    import torch

    import oracle
    from paper_2405_15593_b200 import MicroAdam
    oracle.build()
    d, hp = 36 * BLK + 700, dict(lr=1e-3, window=4)
    th0 = oracle.synth(1, 0, 0, d, dt)
    eng = MicroAdam(d, hp, param_dtype=dt, grad_dtype=dt, value_dtype="bf16")
    orc = oracle.Oracle(th0, hp, param_dtype=dt, value_dtype="bf16")
    p = torch.from_numpy(th0).to(_tdt(dt)).cuda()
    for s in range(1, 9):
        srcs = [torch.from_numpy(oracle.synth(42 + r, s, 0, d, heavy=s % 2 == 0) * (0.5 + r)).to(_tdt(dt)).cuda()
                for r in range(nsrc)]
        out = torch.empty_like(srcs[0])
        eng.step_reduce(p, out, srcs, 1.0 / nsrc, hp["lr"])
        g = _reduce(srcs, 1.0 / nsrc).to(torch.float64).cpu().numpy()
        orc.step(g, hp["lr"])
        torch.cuda.synchronize()
        so = orc.state()
        assert np.array_equal(out.to(torch.float64).cpu().numpy().view(np.uint64), g.view(np.uint64))
        assert np.array_equal(p.to(torch.float64).cpu().numpy().view(np.uint64), so.params.view(np.uint64)), \
            f"θ vs oracle @ {s}"
        eb = eng.error_buffer()
        assert np.array_equal(eb.codes, so.codes), f"EF codes vs oracle @ {s}"
        assert np.array_equal(eb.lo.view(np.uint64), so.lo.view(np.uint64))
        assert np.array_equal(eb.hi.view(np.uint64), so.hi.view(np.uint64))
        win = eng.window()
        for r in range(so.filled):
            assert np.array_equal(win.indices[r], so.win_idx[r]), f"row {r} @ {s}"
            assert np.array_equal(win.values[r].view(np.uint64), so.win_val[r].view(np.uint64))
