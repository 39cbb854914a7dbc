"""Sparse parameter propagation on one GPU.

ma_step_front / ma_scatter_rows / ma_step_stats split the step so that
data-parallel ranks exchange only the new window rows. Checked here:
front(all blocks) + stats is bit-identical to the fused ma_step, and R
simulated ranks (separate whole-vector handles, each running the front on its
block range with only its gradient shard, the stage buffers concatenated as an
all-gather would, rows scattered, stats on each rank's θ replica) reproduce
the unsharded step bit for bit on every replica — θ, window rows, and each
rank's EF blocks.
"""
import numpy as np
import pytest

import oracle
from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

BLK = 4096


def _eng(d, hp, dt="bf16"):
    from paper_2405_15593_b200 import MicroAdam
    return MicroAdam(d, hp, param_dtype=dt, grad_dtype=dt, value_dtype="bf16")


def _dev(x, dt="bf16"):
    import torch
    t = {"bf16": torch.bfloat16, "f32": torch.float32}[dt]
    return torch.from_numpy(np.ascontiguousarray(x, np.float64)).to(t).cuda()


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_front_plus_stats_equals_fused_step(dt):
    import torch
    d, hp = BLK * 24, dict(lr=1e-2, window=6)
    th0 = oracle.synth(1, 0, 0, d, dt)
    fused, split = _eng(d, hp, dt), _eng(d, hp, dt)
    pf, ps = _dev(th0, dt), _dev(th0, dt)
    nb = d // BLK
    stage = split.stage_buffers(nb)
    for s in range(1, 12):
        g = _dev(oracle.synth(42, s, 0, d, dt), dt)
        fused.step(pf, g, 1e-2)
        split.step_front(g, 0, nb, stage)
        split.step_stats(ps, 1e-2)
    torch.cuda.synchronize()
    assert torch.equal(pf, ps)
    assert np.array_equal(fused.error_buffer().codes, split.error_buffer().codes)
    assert np.array_equal(fused.window().indices, split.window().indices)


@pytest.mark.parametrize("world", [2, 3])
def test_simulated_ranks_match_unsharded(world):
    import torch
    from paper_2405_15593_b200 import sharding
    d, hp = BLK * 20, dict(lr=1e-2, window=5)
    nb = d // BLK
    th0 = oracle.synth(1, 0, 0, d)
    ref, pref = _eng(d, hp), _dev(th0)
    ranks = []
    for r in range(world):
        b0, b1, e0, e1 = sharding.partition_blocks(d, BLK, world, r)
        eng = _eng(d, hp)
        ranks.append(dict(eng=eng, b0=b0, b1=b1, e0=e0, e1=e1, p=_dev(th0), stage=eng.stage_buffers(b1 - b0)))
    for s in range(1, 10):
        g = _dev(oracle.synth(42, s, 0, d))
        ref.step(pref, g, 1e-2)
        for rk in ranks:  # each rank sees only its gradient shard
            rk["eng"].step_front(g[rk["e0"]:rk["e1"]].clone(), rk["b0"], rk["b1"], rk["stage"])
        gathered = (torch.cat([rk["stage"][0] for rk in ranks]), torch.cat([rk["stage"][1] for rk in ranks]))
        for rk in ranks:
            rk["eng"].scatter_rows(gathered, 0, nb)
            rk["eng"].step_stats(rk["p"], 1e-2)
    torch.cuda.synchronize()
    codes_ref = ref.error_buffer().codes
    lo_ref = ref.error_buffer().lo.view(np.uint64)
    for rk in ranks:
        assert torch.equal(rk["p"], pref), "θ replica differs"
        assert np.array_equal(rk["eng"].window().indices, ref.window().indices)
        c0, c1 = rk["e0"] // 2, rk["e1"] // 2
        assert np.array_equal(rk["eng"].error_buffer().codes[c0:c1], codes_ref[c0:c1])
        q0, q1 = rk["e0"] // 64, rk["e1"] // 64
        assert np.array_equal(rk["eng"].error_buffer().lo.view(np.uint64)[q0:q1], lo_ref[q0:q1])


def test_split_calls_out_of_order_are_rejected():
    d = BLK * 4
    eng, p = _eng(d, dict(lr=1e-2)), _dev(oracle.synth(1, 0, 0, d))
    with pytest.raises(RuntimeError, match="no ma_step_front"):
        eng.step_stats(p, 1e-2)
    stage = eng.stage_buffers(4)
    with pytest.raises(RuntimeError, match="no ma_step_front"):
        eng.scatter_rows(stage, 0, 4)


@pytest.mark.parametrize("world", [2, 4])
def test_simulated_ranks_match_oracle(world):
    """Sparse propagation across simulated ranks against the composed oracle
    (not against the library's own ma_step): every replica's θ, window rows and
    each rank's EF blocks after every step. Anchors: optim.cpp:183-187 (update
    support ⊆ window rows), window.cpp:28-46."""
    import torch
    from paper_2405_15593_b200 import sharding
    oracle.build()
    d, hp = BLK * 18, dict(lr=1e-2, window=5)
    nb = d // BLK
    th0 = oracle.synth(1, 0, 0, d, "bf16")
    orc = oracle.Oracle(th0, hp, param_dtype="bf16", value_dtype="bf16")
    ranks = []
    for r in range(world):
        b0, b1, e0, e1 = sharding.partition_blocks(d, BLK, world, r)
        eng = _eng(d, hp)
        ranks.append(dict(eng=eng, b0=b0, b1=b1, e0=e0, e1=e1, p=_dev(th0), stage=eng.stage_buffers(b1 - b0)))
    for s in range(1, 11):
        gh = oracle.synth(42, s, 0, d, "bf16", heavy=True)
        g = _dev(gh)
        orc.step(gh, 1e-2)
        for rk in ranks:
            rk["eng"].step_front(g[rk["e0"]:rk["e1"]].clone(), rk["b0"], rk["b1"], rk["stage"])
        gathered = (torch.cat([rk["stage"][0] for rk in ranks]), torch.cat([rk["stage"][1] for rk in ranks]))
        for rk in ranks:
            rk["eng"].scatter_rows(gathered, 0, nb)
            rk["eng"].step_stats(rk["p"], 1e-2)
        torch.cuda.synchronize()
        so = orc.state()
        for rk in ranks:
            got = rk["p"].to(torch.float64).cpu().numpy()
            assert np.array_equal(got.view(np.uint64), so.params.view(np.uint64)), f"θ replica vs oracle @ {s}"
            win = rk["eng"].window()
            for r in range(so.filled):
                assert np.array_equal(win.indices[r], so.win_idx[r]), f"row {r} @ {s}"
            codes, lo, _ = rk["eng"].error_buffer_blocks(rk["b0"], rk["b1"])
            c0, c1 = rk["e0"] // 2, rk["e1"] // 2
            assert np.array_equal(codes, so.codes[c0:c1]), f"EF codes of rank blocks @ {s}"
            assert np.array_equal(lo.view(np.uint64), so.lo[rk["e0"] // 64: rk["e1"] // 64].view(np.uint64))
