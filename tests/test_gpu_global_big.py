"""Global Top-K mode (the reference's default, topk_global compress.cpp:66-71)
at d > 2^32 on the device: int64 window indices past 2^31 and 2^32.

A 4.3-billion-element bf16 vector is too large for the CPU oracle, so the
gradient is built to make the selection known: the ma_synth stream
(|g| < 4) plus k spikes of magnitude >= 64 at fixed positions straddling 2^31,
2^32 and the tail. Every step then selects exactly the spikes, and:
* the window row (int64 global indices, bf16 values) equals the spike
  positions and rn_bf16(a) with a = g + decode(EF) computed on the host from
  the device's previous (already checked) codes of those buckets;
* the EF codes and (lo, hi) of every 4096-chunk holding a spike, and of the
  last (partial) chunk, are bit-exact against the oracle's
  QuantizedErrorBuffer::encode (quantize.cpp:142-162) of the residual slice;
* θ at the spikes equals a composed-oracle run on just those coordinates (the
  same rows, stamps and weights: window.cpp:28-46, optim.cpp:183-187), and θ
  next to them is untouched.
"""
import ctypes as C

import numpy as np
import pytest

import oracle
from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

CH = 4096


def _bf16_bits_to_f64(u16):
    return (np.asarray(u16, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def test_global_mode_beyond_2_pow_32():
    import torch

    import paper_2405_15593_b200 as ma
    d = 2 ** 32 + 2 * CH + 200
    fixed = [7, 3 * CH + 64, 2 ** 31 - 3, 2 ** 31, 2 ** 31 + CH + 1, 2 ** 32 - 1, 2 ** 32, 2 ** 32 + 5, d - 1]
    rng = np.random.default_rng(5)
    pos = np.unique(np.concatenate([fixed, rng.integers(0, d, 15)]))
    k = int(pos.size)
    hp = dict(lr=1e-2, window=3, k=k)
    eng = ma.MicroAdam(d, hp, param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16", blockwise=False)
    L = ma.lib()
    s = torch.cuda.current_stream().cuda_stream
    theta = torch.empty(d, dtype=torch.bfloat16, device="cuda")
    g = torch.empty(d, dtype=torch.bfloat16, device="cuda")
    ma._capi.check(L.ma_fill_synthetic(theta.data_ptr(), 2, d, 1, 0, 0, 0, s))
    th0_sp = theta[torch.from_numpy(pos).cuda()].view(torch.int16).cpu().numpy()
    small = oracle.Oracle(_bf16_bits_to_f64(th0_sp), dict(hp, block=k), param_dtype="bf16", value_dtype="bf16")
    chunks = sorted(set((pos // CH).tolist()) | {(d - 1) // CH})
    prev = {c: (np.zeros(min(CH, d - c * CH) // 2 + (min(CH, d - c * CH) & 1), np.uint8),
                np.zeros(CH // 64), np.zeros(CH // 64)) for c in chunks}
    OL = oracle.oracle_lib()
    for step in range(1, 5):
        ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), 2, d, 42, step, 0, 0, s))
        spike = np.array([(64 + j + step) * (-1) ** j for j in range(k)], np.float64)  # bf16-exact
        g[torch.from_numpy(pos).cuda()] = torch.from_numpy(spike).to(torch.bfloat16).cuda()
        eng.step(theta, g, hp["lr"])
        eng.synchronize()
        # a at the spikes: g + decode(previous EF of their buckets)
        a_sp = np.empty(k)
        for c in chunks:
            n = min(CH, d - c * CH)
            gs = oracle.synth(42, step, c * CH, n, "bf16")
            inside = (pos >= c * CH) & (pos < c * CH + n)
            gs[pos[inside] - c * CH] = spike[inside]
            codes0, lo0, hi0 = prev[c]
            e = np.zeros(n)
            if step > 1:
                nb = (n + 63) // 64
                OL.mo_decode(np.ascontiguousarray(codes0), np.ascontiguousarray(lo0[:nb]),
                             np.ascontiguousarray(hi0[:nb]), n, 4, 64, e)
            a = gs + e
            a_sp[inside] = a[pos[inside] - c * CH]
            r = a.copy()
            r[pos[inside] - c * CH] = 0.0  # the spikes are the selection
            # device EF of the chunk vs the oracle's encode of the residual
            nb = (n + 63) // 64
            codes = np.zeros((n + 1) // 2, np.uint8)
            lo, hi = np.zeros(nb), np.zeros(nb)
            L.ma_read_error_buffer_blocks(eng._h, c, c + 1, codes.ctypes.data_as(C.c_void_p),
                                          lo.ctypes.data_as(C.c_void_p), hi.ctypes.data_as(C.c_void_p))
            ocodes, olo, ohi = np.zeros((n + 1) // 2, np.uint8), np.zeros(nb), np.zeros(nb)
            OL.mo_encode(np.ascontiguousarray(r), n, 4, 64, ocodes, olo, ohi)
            assert np.array_equal(codes, ocodes), f"EF codes of chunk {c} @ step {step}"
            assert np.array_equal(lo.view(np.uint64), olo.view(np.uint64)), f"lo of chunk {c} @ step {step}"
            assert np.array_equal(hi.view(np.uint64), ohi.view(np.uint64)), f"hi of chunk {c} @ step {step}"
            prev[c] = (codes, np.pad(lo, (0, CH // 64 - nb)), np.pad(hi, (0, CH // 64 - nb)))
        # window row: int64 indices past 2^31 / 2^32, values rn_bf16(a)
        head = eng.counters()[1]
        slot = (head + hp["window"] - 1) % hp["window"]
        idx = np.zeros(k, np.int64)
        val = np.zeros(k)
        ma._capi.check(L.ma_read_window_row(eng._h, slot, idx.ctypes.data_as(C.c_void_p),
                                            val.ctypes.data_as(C.c_void_p)))
        assert np.array_equal(idx, pos), f"selection @ step {step}"
        want = np.array([OL.mo_bf16_round(x) for x in a_sp])
        assert np.array_equal(val.view(np.uint64), want.view(np.uint64)), f"window values @ step {step}"
        # θ at the spikes vs the composed oracle on those coordinates
        small.step(a_sp, hp["lr"])
        got = _bf16_bits_to_f64(theta[torch.from_numpy(pos).cuda()].view(torch.int16).cpu().numpy().view(np.uint16))
        assert np.array_equal(got.view(np.uint64), small.state().params.view(np.uint64)), f"θ @ step {step}"
    # neighbours of the spikes never entered the window: θ unchanged
    for p0 in (2 ** 31 + 1, 2 ** 32 + 1, d - 2):
        cur = theta[p0: p0 + 1].view(torch.int16).cpu().numpy().view(np.uint16)
        want0 = oracle.synth(1, 0, p0, 1, "bf16")
        assert _bf16_bits_to_f64(cur)[0] == want0[0]
