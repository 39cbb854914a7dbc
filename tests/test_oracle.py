"""Pin the CPU oracle (oracle/microadam_oracle.c) before trusting it.

1. The reference's own known-answer tests, transcribed from
   /root/reference/proj/tests/{test_compress,test_quantize,test_window,test_optim}.cpp
   (file:line cited per test), run against the C restatement.
2. tests/golden/*.npz — produced by the UNMODIFIED reference
   (oracle/make_golden.py) — replayed through the restatement: every step's
   state digest must match.
3. Where oracle/_ref is built (this container), randomized live differential
   runs of restatement vs reference.
"""
import glob
import hashlib
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def L():
    oracle.build()
    return oracle.oracle_lib()


def topk_global(L, x, k):
    x = np.asarray(x, np.float64)
    idx = np.zeros(k, np.int64)
    val = np.zeros(k)
    n = L.mo_topk_global(x, x.size, k, idx, val)
    assert n == k
    return idx, val


def topk_blockwise(L, x, block, kb):
    x = np.asarray(x, np.float64)
    cap = x.size
    idx = np.zeros(cap, np.int64)
    val = np.zeros(cap)
    n = L.mo_topk_blockwise(x, x.size, block, kb, idx, val)
    return idx[:n], val[:n]


# ---- compress (test_compress.cpp) -------------------------------------------
def test_topk_global_kat(L):  # test_compress.cpp:38-50
    idx, val = topk_global(L, [3.0, -7.0, 1.0, 0.5], 2)
    assert idx.tolist() == [0, 1] and val.tolist() == [3.0, -7.0]
    idx, val = topk_global(L, [5.0, 0.0, 0.0], 3)
    assert idx.tolist() == [0, 1, 2] and val.tolist() == [5.0, 0.0, 0.0]
    idx, _ = topk_global(L, [2.0, -2.0, 2.0], 1)
    assert idx.tolist() == [0]


def test_topk_global_sort_oracle(L):  # test_compress.cpp:52-63
    rng = np.random.default_rng(11)
    for _ in range(200):
        d = 1 + int(rng.integers(64))
        x = rng.standard_normal(d)
        k = 1 + int(rng.integers(d))
        order = sorted(range(d), key=lambda i: (-abs(x[i]), i))[:k]
        idx, val = topk_global(L, x, k)
        assert idx.tolist() == sorted(order)
        assert np.array_equal(val, x[idx])


def test_topk_blockwise_kat(L):  # test_compress.cpp:71-82, 97-113
    idx, _ = topk_blockwise(L, [3.0, -7.0, 1.0, 0.5], 2, 1)
    assert idx.tolist() == [1, 2]
    idx, _ = topk_blockwise(L, np.ones(8), 4, 1)
    assert idx.tolist() == [0, 4]
    idx, _ = topk_blockwise(L, np.arange(1.0, 11.0), 4, 3)
    assert idx.size == 3 + 3 + 2 and (idx < 10).all()
    assert L.mo_per_block_k(10, 0.25) == 3
    assert L.mo_per_block_k(2, 0.5) == 1


def test_single_block_equals_global(L):  # test_compress.cpp:84-95
    rng = np.random.default_rng(12)
    for _ in range(100):
        d = 2 + int(rng.integers(40))
        x = rng.standard_normal(d)
        k = 1 + int(rng.integers(d))
        a = topk_blockwise(L, x, d, k)
        b = topk_global(L, x, k)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ---- quantize (test_quantize.cpp) --------------------------------------------
def qparams(L, x):
    import ctypes as C
    lo, hi = C.c_double(), C.c_double()
    x = np.asarray(x, np.float64)
    L.mo_quant_params(x, x.size, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def test_quant_params_kat(L):  # test_quantize.cpp:28-41
    lo, hi = qparams(L, [0.0, 7.4, 15.0])
    assert (lo, hi) == (0.0, 15.0) and L.mo_level(lo, hi, 4) == 1.0
    lo, hi = qparams(L, [3.5, 3.5, 3.5])
    assert lo == hi and L.mo_level(lo, hi, 4) == 0.0
    lo, hi = qparams(L, [-1.0, 1.0])
    assert L.mo_level(lo, hi, 1) == 2.0


def test_quantize_nearest_kat(L):  # test_quantize.cpp:43-55
    lo, hi = qparams(L, [0.0, 7.4, 15.0])
    lvl = L.mo_level(lo, hi, 4)
    assert [L.mo_quantize_nearest(x, lo, lvl, 4) for x in (0.0, 7.4, 15.0)] == [0, 7, 15]
    assert L.mo_quantize_nearest(lo + lvl / 2.0, lo, lvl, 4) == 1  # half-up
    assert L.mo_quantize_nearest(2.0, 2.0, 0.0, 4) == 0  # flat grid


def test_pack_kat(L):  # test_quantize.cpp:137-154
    out = np.zeros(1, np.uint8)
    L.mo_pack(np.array([1, 2], np.uint32), 2, 4, out)
    assert out.tolist() == [0x21]
    out = np.zeros(2, np.uint8)
    L.mo_pack(np.array([15, 15, 15], np.uint32), 3, 4, out)
    assert out.tolist() == [0xFF, 0x0F]
    back = np.zeros(3, np.uint32)
    L.mo_unpack(out, 3, 4, back)
    assert back.tolist() == [15, 15, 15]
    rng = np.random.default_rng(35)
    for _ in range(300):
        bits = 1 + int(rng.integers(8))
        n = 1 + int(rng.integers(77))
        codes = (rng.integers(0, 2 ** 32, n, dtype=np.uint64) & ((1 << bits) - 1)).astype(np.uint32)
        buf = np.zeros((n * bits + 7) // 8, np.uint8)
        L.mo_pack(codes, n, bits, buf)
        back = np.zeros(n, np.uint32)
        L.mo_unpack(buf, n, bits, back)
        assert np.array_equal(back, codes)


def encode(L, x, bucket, bits=4):
    x = np.asarray(x, np.float64)
    nb = (x.size + bucket - 1) // bucket
    codes = np.zeros((x.size * bits + 7) // 8, np.uint8)
    lo, hi = np.zeros(nb), np.zeros(nb)
    L.mo_encode(x, x.size, bits, bucket, codes, lo, hi)
    out = np.zeros(x.size)
    L.mo_decode(codes, lo, hi, x.size, bits, bucket, out)
    return codes, lo, hi, out


def test_error_buffer_zeros_and_bucket_local(L):  # test_quantize.cpp:194-220
    codes, lo, hi, out = encode(L, np.zeros(100), 64)
    assert codes.size == 50 and lo.size == 2 and (out == 0).all()
    rng = np.random.default_rng(38)
    for _ in range(50):
        d = 1 + int(rng.integers(300))
        bucket = 1 + int(rng.integers(80))
        x = rng.standard_normal(d) * 2.0
        codes, lo, hi, back = encode(L, x, bucket)
        assert codes.size == (d * 4 + 7) // 8 and lo.size == (d + bucket - 1) // bucket
        for i in range(d):
            b = i // bucket
            lvl = L.mo_level(lo[b], hi[b], 4)
            assert abs(back[i] - x[i]) <= lvl / 2 + 1e-12 * (abs(hi[b]) + abs(lo[b]) + 1)


def test_bucket_of_two_is_lossless(L):  # test_quantize.cpp:222-227
    x = np.array([3.25, -1.5, 0.75, 2.125])
    assert np.array_equal(encode(L, x, 2)[3], x)


# ---- window (test_window.cpp) ------------------------------------------------
def adam_stats(L, rows_idx, rows_val, stamps, step, dim, beta, square):
    m, rw = rows_idx.shape
    z = np.zeros(dim)
    filled = min(step, m)
    L.mo_adam_stats(np.ascontiguousarray(rows_idx, np.int64), np.ascontiguousarray(rows_val),
                    np.ascontiguousarray(stamps, np.int64), m, rw, filled, step, dim, beta,
                    int(square), z)
    return z


def test_two_step_moment_kat(L):  # test_window.cpp:67-76
    z = adam_stats(L, np.array([[0], [0]]), np.array([[1.0], [2.0]]), np.array([1, 2]), 2, 1, 0.9,
                   False)
    assert z[0] == 0.29 / 0.19 or abs(z[0] - 0.29 / 0.19) <= 1e-15 * z[0]
    assert abs(z[0] - 1.526316) <= 1e-6


def test_single_row_and_square_kat(L):  # test_window.cpp:78-91
    z = adam_stats(L, np.array([[0, 2]] + [[0, 0]] * 4), np.array([[4.0, -1.5]] + [[0, 0]] * 4),
                   np.array([1, 0, 0, 0, 0]), 1, 3, 0.9, False)
    assert z.tolist() == [4.0, 0.0, -1.5]
    z = adam_stats(L, np.array([[3], [0]]), np.array([[-2.0], [0.0]]), np.array([1, 0]), 1, 5, 0.5,
                   True)
    assert z[3] == 4.0 and (z[[0, 1, 2, 4]] == 0).all()


def test_window_matches_dense_ema(L):  # test_window.cpp:114-162 (dense rows, t <= m)
    rng = np.random.default_rng(41)
    for _ in range(60):
        d = 1 + int(rng.integers(16))
        m = 1 + int(rng.integers(8))
        t = 1 + int(rng.integers(m))
        beta = 0.5 + 0.49 * rng.random()
        hist = rng.standard_normal((t, d))
        idx = np.tile(np.arange(d), (m, 1))
        val = np.zeros((m, d))
        val[:t] = hist
        stamps = np.zeros(m, np.int64)
        stamps[:t] = np.arange(1, t + 1)
        for square in (False, True):
            got = adam_stats(L, idx, val, stamps, t, d, beta, square)
            z = np.zeros(d)
            for g in hist:
                z = beta * z + (1 - beta) * (g * g if square else g)
            want = z / (1 - beta ** t)
            assert np.all(np.abs(got - want) <= 1e-12 * np.maximum(1, np.abs(want)))


# ---- optimizer step (test_optim.cpp) -------------------------------------------
def test_blockwise_step_kat():  # test_optim.cpp:265-274
    o = oracle.Oracle(np.zeros(8), dict(density=0.25, block=4, lr=1e-2))
    o.step(np.array([9.0, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0]))
    assert o.state().last_idx.tolist() == [0, 7]


def test_update_support_within_window():  # test_optim.cpp:239-263 (blockwise variant)
    rng = np.random.default_rng(66)
    o = oracle.Oracle(np.zeros(20), dict(k=2, window=3, lr=1e-2, block=20))
    for _ in range(30):
        before = o.state().params.copy()
        rep = o.step(rng.standard_normal(20))
        st = o.state()
        assert rep["update_nnz"] <= 3 * 2
        moved = np.flatnonzero(st.params != before)
        in_window = set(st.win_idx[: st.filled].ravel().tolist())
        assert set(moved.tolist()) <= in_window
        assert moved.size == rep["update_nnz"]


def test_bf16_round_rule():
    L = oracle.oracle_lib()
    # ties to even at the bf16 mantissa boundary, from a double directly
    one = 1.0
    ulp = 2.0 ** -7
    assert L.mo_bf16_round(one + ulp / 2) == one                 # tie -> even (1.0)
    assert L.mo_bf16_round(one + 3 * ulp / 2) == one + 2 * ulp   # tie -> even (up)
    assert L.mo_bf16_round(one + ulp / 2 + 2.0 ** -40) == one + ulp  # above tie: up
    assert L.mo_bf16_round(3.0e38 * 10) == math.inf
    assert L.mo_bf16_round(2.0 ** -133) == 2.0 ** -133           # bf16 subnormal
    assert L.mo_bf16_round(-2.0 ** -135) == 0.0 and math.copysign(1, L.mo_bf16_round(-2.0 ** -135)) < 0
    # double rounding trap: a double just above a bf16 tie that rounds to the tie in fp32
    x = 1.0 + ulp / 2 + 2.0 ** -30
    assert np.float32(x) == np.float32(1.0 + ulp / 2)  # fp32 loses the tiebreaker bit
    assert L.mo_bf16_round(x) == one + ulp             # direct rounding keeps it


# ---- golden fixtures (unmodified reference) ------------------------------------
def _digest(st):
    h = hashlib.sha256()
    for a in (st.last_idx, st.last_val, st.codes, st.lo, st.hi, st.params):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def golden_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))


def golden_grads(meta, step):
    if meta["generator"] == "zeros":
        return np.zeros(meta["dim"])
    return oracle.synth(42, step, 0, meta["dim"], meta["grad_dtype"],
                        levels=meta["generator"] == "levels")


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_replays_golden(path):
    z = np.load(path)
    meta = json.loads(str(z["meta"]))
    hp = dict(meta["hp"])
    if not meta["blockwise"]:
        hp["block"] = meta["dim"]
    o = oracle.Oracle(oracle.synth(1, 0, 0, meta["dim"], meta["grad_dtype"]), hp)
    for s in range(1, meta["steps"] + 1):
        rep = o.step(golden_grads(meta, s))
        st = o.state()
        assert _digest(st) == str(z["digests"][s - 1]), f"step {s}"
        r = z["reports"][s - 1]
        assert [rep["grad_norm"], rep["error_norm"], rep["empirical_q"], rep["update_nnz"]] == list(r)
    st = o.state()
    assert np.array_equal(st.win_idx[: st.filled], z["win_idx"][: st.filled])
    assert np.array_equal(st.win_val[: st.filled], z["win_val"][: st.filled])
    assert (st.step, st.head, st.filled) == (int(z["step"]), int(z["head"]), int(z["filled"]))


def test_golden_fixtures_present():
    assert len(golden_cases()) >= 6


# ---- live differential vs the compiled reference -------------------------------
@pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(6))
def test_oracle_matches_reference_random_configs(seed):
    rng = np.random.default_rng(100 + seed)
    d = int(rng.integers(5, 20_000))
    block = int(rng.choice([4, 16, 64, 256, 1000, 4096]))
    bucket = int(rng.choice([1, 2, 3, 16, 64, 100]))
    hp = dict(block=block, bucket=bucket, window=int(rng.integers(1, 12)),
              density=float(rng.choice([0.001, 0.01, 0.05, 0.3])), lr=1e-2)
    theta0 = rng.standard_normal(d)
    o, r = oracle.Oracle(theta0, hp), oracle.Reference(theta0, hp)
    for s in range(1, 8):
        g = oracle.synth(seed, s, 0, d, "f32", levels=bool(seed % 2))
        assert o.step(g) == r.step(g)
        so, sr = o.state(), r.state()
        assert np.array_equal(so.params.view(np.uint64), sr.params.view(np.uint64))
        assert np.array_equal(so.codes, sr.codes)
        assert np.array_equal(so.lo.view(np.uint64), sr.lo.view(np.uint64))
        assert np.array_equal(so.last_idx, sr.last_idx)


@pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("bits", [1, 3, 8, 12, 16, 23, 24])
def test_oracle_matches_reference_code_widths(bits):
    # HyperParams::bits in [1, 24] (optim.cpp:12): bit stream + max_code = 2^bits - 1
    rng = np.random.default_rng(bits)
    d = 9_001
    hp = dict(block=1000, bucket=8, window=3, lr=1e-2, bits=bits)
    theta0 = rng.standard_normal(d)
    o, r = oracle.Oracle(theta0, hp), oracle.Reference(theta0, hp)
    for s in range(1, 6):
        g = oracle.synth(7, s, 0, d, "f32")
        assert o.step(g) == r.step(g)
        so, sr = o.state(), r.state()
        assert np.array_equal(so.params.view(np.uint64), sr.params.view(np.uint64))
        assert np.array_equal(so.codes, sr.codes)
        assert np.array_equal(so.lo.view(np.uint64), sr.lo.view(np.uint64))
