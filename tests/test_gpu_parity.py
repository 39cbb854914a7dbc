"""Parity of the CUDA step (through the C ABI) against the CPU checkers.

Bar (north star): Top-K indices, EF codes and bucket (lo, hi)
bit-exact against the reference for every dtype; θ and window values
bit-exact against the composed oracle (reference algorithm with the device's
storage roundings), and bit-exact against the UNMODIFIED reference in fp64
mode. Reports (norms) within 1e-12 relative; update_nnz exact.
"""
import numpy as np
import pytest

import oracle
from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

TORCH_DT = {}


def _torch():
    import torch
    if not TORCH_DT:
        TORCH_DT.update({"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16})
    return torch


def _bits(x):
    return np.asarray(x, np.float64).view(np.uint64)


def _dev(x, dt):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(x, np.float64)).to(TORCH_DT[dt]).cuda()


def _host(t):
    torch = _torch()
    return t.detach().to(torch.float64).cpu().numpy()


KERNELS = {"fast": {}, "warp_exact": {"MA_WARP_EXACT": "1"}, "fast_cta": {"MA_FAST_CTA": "1"},
           "generic": {"MA_FORCE_GENERIC": "1"}}


def make_engine(kernel, *args, **kw):
    """Create a MicroAdam engine with the kernel family selected at ma_create time."""
    import os
    from paper_2405_15593_b200 import MicroAdam
    saved = {k: os.environ.get(k) for k in ("MA_FAST_CTA", "MA_FORCE_GENERIC", "MA_WARP_EXACT")}
    for k in saved:
        os.environ.pop(k, None)
    os.environ.update(KERNELS[kernel])
    try:
        return MicroAdam(*args, **kw)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def run_parity(d, hp, *, gdt="f32", pdt="f32", vdt="bf16", steps=12, levels=False, seed=42,
               grad_fn=None, check_reference=None, lr=None, report_every=0, kernel="fast",
               theta0=None, check_every=1):
    torch = _torch()
    oracle.build()
    lr = hp.get("lr", 1e-3) if lr is None else lr
    if theta0 is None:
        theta0 = oracle.synth(1, 0, 0, d, pdt)
    theta0 = _host(_dev(np.asarray(theta0, np.float64), pdt))  # representable in the param dtype
    orc = oracle.Oracle(theta0, hp, param_dtype=pdt, value_dtype=vdt)
    ref = None
    if check_reference is None:
        check_reference = pdt == "f64" and vdt == "f64" and oracle.reference_available()
    if check_reference:
        ref = oracle.Reference(theta0, hp)
    eng = make_engine(kernel, d, hp, param_dtype=pdt, grad_dtype=gdt, value_dtype=vdt)
    params = _dev(theta0, pdt)
    for s in range(1, steps + 1):
        g = grad_fn(s) if grad_fn else oracle.synth(seed, s, 0, d, gdt, levels=levels)
        g = _host(_dev(np.asarray(g, np.float64), gdt))  # the values the device sees
        want_rep = bool(report_every) and s % report_every == 0
        rep = eng.step(params, _dev(g, gdt), lr, report=want_rep)
        orep = orc.step(g, lr)
        if ref is not None:
            ref.step(g)
        if s % check_every and s != steps:
            continue
        torch.cuda.synchronize()
        eng.synchronize()
        so = orc.state()
        win = eng.window()
        eb = eng.error_buffer()
        step, head, filled, stamps = eng.counters()
        assert (step, head, filled) == (so.step, so.head, so.filled), f"counters @ step {s}"
        assert np.array_equal(stamps, so.stamps)
        slot = (head + orc.m - 1) % orc.m
        assert np.array_equal(win.indices[slot], so.last_idx), f"Top-K indices differ @ step {s}"
        assert np.array_equal(eb.codes, so.codes), f"EF codes differ @ step {s}"
        assert np.array_equal(_bits(eb.lo), _bits(so.lo)), f"EF lo differ @ step {s}"
        assert np.array_equal(_bits(eb.hi), _bits(so.hi)), f"EF hi differ @ step {s}"
        for r in range(filled):
            assert np.array_equal(win.indices[r], so.win_idx[r]), f"window row {r} idx @ {s}"
            assert np.array_equal(_bits(win.values[r]), _bits(so.win_val[r])), f"row {r} val @ {s}"
        got = _host(params)
        bad = np.flatnonzero(_bits(got) != _bits(so.params))
        assert bad.size == 0, f"θ differs @ step {s} at {bad[:8]}: {got[bad[:4]]} vs {so.params[bad[:4]]}"
        if want_rep:
            for k in ("grad_norm", "error_norm", "empirical_q"):
                a, b = getattr(rep, k), orep[k]
                assert abs(a - b) <= 1e-12 * max(abs(b), 1e-300), (k, a, b)
            assert rep.update_nnz == orep["update_nnz"]
        if ref is not None:
            sr = ref.state()
            assert np.array_equal(_bits(sr.params), _bits(got)), f"θ vs unmodified reference @ {s}"
            assert np.array_equal(sr.codes, eb.codes)
            assert np.array_equal(sr.last_idx, win.indices[slot])
    return eng, orc


@pytest.mark.parametrize("kernel", sorted(KERNELS))
def test_default_config_1m_fp32_bf16_window(kernel):
    # SURVEY config 1 shape (1M params, density 1%, m=10, 4-bit EF, B_d 4096, B_q 64).
    run_parity(1_000_000, dict(lr=1e-3), gdt="f32", pdt="f32", vdt="bf16", steps=20,
               report_every=5, kernel=kernel)


@pytest.mark.parametrize("kernel", sorted(KERNELS))
def test_fp64_mode_bit_exact_vs_unmodified_reference(kernel):
    run_parity(200_000, dict(lr=1e-3), gdt="f64", pdt="f64", vdt="f64", steps=15,
               check_reference=oracle.reference_available(), kernel=kernel)


def test_bf16_params_and_grads():
    run_parity(300_000, dict(lr=1e-3), gdt="bf16", pdt="bf16", vdt="bf16", steps=12)


def test_fp32_params_fp64_window():
    run_parity(100_000, dict(lr=1e-2), gdt="f32", pdt="f32", vdt="f64", steps=12)


def test_fp32_window_values():
    run_parity(100_000, dict(lr=1e-2), gdt="bf16", pdt="f32", vdt="f32", steps=8)


@pytest.mark.parametrize("d,block,bucket,density,m", [
    (4099, 512, 16, 0.01, 3),      # short tail block, smaller buckets
    (37, 8, 4, 0.25, 2),           # odd d, odd tail
    (10_000, 4096, 64, 0.05, 20),  # m=20, 5% density
    (50_000, 4096, 64, 0.001, 5),  # 0.1% -> k_b = 5
    (20_000, 1000, 8, 0.02, 4),    # block not a power of two
    (8192 * 3 + 5, 8192, 64, 0.01, 10),  # the 8192 variant + 5-element tail
    (130, 128, 64, 0.5, 1),        # m = 1
    (8, 4, 2, 0.25, 10),           # test_optim.cpp:265-274 shape
    (1, 4096, 64, 0.01, 3),        # d = 1: block = 1, the element is always selected
    (3, 2, 1, 0.5, 2),             # bucket 1, ragged last block
])
@pytest.mark.parametrize("kernel", ["fast", "generic"])
def test_shapes(d, block, bucket, density, m, kernel):
    hp = dict(block=block, bucket=bucket, density=density, window=m, lr=1e-2)
    run_parity(d, hp, gdt="f64", pdt="f64", vdt="f64", steps=m + 4, kernel=kernel)


@pytest.mark.parametrize("kernel", sorted(KERNELS))
def test_tie_heavy_levels(kernel):
    # 16 grad levels: many exact |a| ties; index order must decide.
    run_parity(40_000, dict(lr=1e-2), gdt="f32", pdt="f32", vdt="bf16", steps=10, levels=True,
               kernel=kernel)


@pytest.mark.parametrize("kernel", sorted(KERNELS))
def test_zero_gradient_degenerate_buckets(kernel):
    # all-zero gradients: every |a| ties, every bucket lo == hi (level 0).
    run_parity(20_000, dict(lr=1e-2), gdt="f32", pdt="f32", vdt="bf16", steps=6,
               grad_fn=lambda s: np.zeros(20_000), kernel=kernel)


@pytest.mark.parametrize("bucket", [16, 32])
def test_fast_kernel_small_buckets(bucket):
    run_parity(70_000, dict(lr=1e-2, bucket=bucket), gdt="bf16", pdt="bf16", vdt="bf16", steps=8)


def test_distribution_shift_and_threshold_recovery():
    # scale jumps by 2^20 between steps: the carried Top-K threshold is wrong
    # in both directions and the exact fallback must take over.
    scales = [1.0, 2.0 ** 20, 2.0 ** 20, 2.0 ** -20, 1.0, 1.0, 3.0, 1.0]
    run_parity(60_000, dict(lr=1e-2), gdt="f64", pdt="f64", vdt="f64", steps=len(scales),
               grad_fn=lambda s: oracle.synth(9, s, 0, 60_000) * scales[s - 1])


def test_sparse_spiky_gradients():
    # mostly zeros with a few spikes per block: exercises the radix fallback.
    rng = np.random.default_rng(3)

    def g(s):
        x = np.zeros(30_000)
        idx = rng.choice(30_000, 200, replace=False)
        x[idx] = np.round(rng.standard_normal(200) * 1e3) / 8
        return x
    run_parity(30_000, dict(lr=1e-2), gdt="f64", pdt="f64", vdt="f64", steps=8, grad_fn=g)


def test_scales_tiny_and_huge():
    for scale in (2.0 ** -60, 2.0 ** 40):
        run_parity(9_000, dict(lr=1e-3), gdt="f64", pdt="f64", vdt="bf16", steps=5,
                   grad_fn=lambda s, sc=scale: oracle.synth(7, s, 0, 9_000) * sc)


def test_global_mode_small_d():
    # blockwise=false (the reference default) == one block spanning d when d <= 8192.
    from paper_2405_15593_b200 import MicroAdam
    torch = _torch()
    d, hp = 3000, dict(k=30, lr=1e-2, window=4)
    theta0 = oracle.synth(1, 0, 0, d)
    ref = oracle.Reference(theta0, hp, blockwise=False) if oracle.reference_available() else None
    orc = oracle.Oracle(theta0, dict(hp, block=d))
    eng = MicroAdam(d, hp, param_dtype="f64", grad_dtype="f64", value_dtype="f64", blockwise=False)
    params = _dev(theta0, "f64")
    for s in range(1, 8):
        g = oracle.synth(42, s, 0, d)
        eng.step(params, _dev(g, "f64"), 1e-2)
        orc.step(g, 1e-2)
        torch.cuda.synchronize()
        so = orc.state()
        assert np.array_equal(_bits(_host(params)), _bits(so.params))
        if ref is not None:
            ref.step(g)
            assert np.array_equal(_bits(ref.state().params), _bits(so.params))


def test_host_dropin_matches_reference():
    """paper_2405_15593_b200.MicroAdamOptimizer is a drop-in for the reference class."""
    from paper_2405_15593_b200 import MicroAdamOptimizer
    d, hp = 50_000, dict(lr=1e-2, window=4)
    theta0 = oracle.synth(1, 0, 0, d)
    opt = MicroAdamOptimizer(theta0, hp, blockwise=True)
    orc = oracle.Oracle(theta0, hp)
    ref = oracle.Reference(theta0, hp) if oracle.reference_available() else None
    assert opt.name() == "microadam"
    for s in range(1, 9):
        g = oracle.synth(42, s, 0, d)
        rep = opt.step(g)
        orep = orc.step(g)
        so = orc.state()
        assert np.array_equal(_bits(opt.params()), _bits(so.params))
        assert np.array_equal(opt.last_selection().indices, so.last_idx)
        assert np.array_equal(_bits(opt.last_selection().values), _bits(so.last_val))
        assert np.array_equal(_bits(opt.error_vector()), _bits(_decode(so, hp)))
        assert rep.update_nnz == orep["update_nnz"]
        assert opt.step_count() == s
        if ref is not None:
            rrep = ref.step(g)
            assert np.array_equal(_bits(ref.state().params), _bits(opt.params()))
            assert abs(rep.grad_norm - rrep["grad_norm"]) <= 1e-12 * rrep["grad_norm"]
    with pytest.raises(ValueError):
        opt.step(np.zeros(d - 1))


def _decode(so, hp):
    bucket = hp.get("bucket", 64)
    d = so.params.size
    codes = np.empty(so.codes.size * 2, np.uint8)
    codes[0::2] = so.codes & 15
    codes[1::2] = so.codes >> 4
    c = codes[:d].astype(np.float64)
    b = np.arange(d) // bucket
    lvl = np.where(so.lo == so.hi, 0.0, (so.hi - so.lo) / 15.0)
    return c * lvl[b] + so.lo[b]


def test_nonfinite_strict_rejects_before_mutation():
    from paper_2405_15593_b200 import InvalidArgument, MicroAdam
    torch = _torch()
    d = 10_000
    eng = MicroAdam(d, dict(lr=1e-2), param_dtype="f32", grad_dtype="f32", finite_mode="strict")
    params = _dev(oracle.synth(1, 0, 0, d, "f32"), "f32")
    eng.step(params, _dev(oracle.synth(42, 1, 0, d, "f32"), "f32"), 1e-2)
    torch.cuda.synchronize()
    before = (_host(params).copy(), eng.error_buffer().codes.copy(), eng.counters()[0])
    g = oracle.synth(42, 2, 0, d, "f32")
    g[1234] = np.nan
    with pytest.raises(InvalidArgument):
        eng.step(params, _dev(g, "f32"), 1e-2)
    assert np.array_equal(_host(params), before[0])
    assert np.array_equal(eng.error_buffer().codes, before[1])
    assert eng.counters()[0] == before[2]


def test_nonfinite_flag_mode_reports_at_sync():
    from paper_2405_15593_b200 import InvalidArgument, MicroAdam
    d = 10_000
    eng = MicroAdam(d, dict(lr=1e-2), param_dtype="f32", grad_dtype="f32", finite_mode="flag")
    params = _dev(oracle.synth(1, 0, 0, d, "f32"), "f32")
    g = oracle.synth(42, 1, 0, d, "f32")
    g[7] = np.inf
    eng.step(params, _dev(g, "f32"), 1e-2)
    with pytest.raises(InvalidArgument):
        eng.synchronize()
    eng.synchronize()  # flag cleared


def test_block_sharding_matches_unsharded():
    """Block-aligned shards reproduce the unsharded step bit-for-bit."""
    from paper_2405_15593_b200 import MicroAdam
    from paper_2405_15593_b200.sharding import partition_blocks
    torch = _torch()
    d, hp = 100_003, dict(lr=1e-2, window=5)
    theta0 = oracle.synth(1, 0, 0, d, "f32")
    full = MicroAdam(d, hp, param_dtype="f32", grad_dtype="f32", value_dtype="bf16")
    p_full = _dev(theta0, "f32")
    lay = full.layout
    shards = []
    for rank in range(3):
        b0, b1, e0, e1 = partition_blocks(d, lay.block, 3, rank)
        eng = MicroAdam(d, hp, param_dtype="f32", grad_dtype="f32", value_dtype="bf16",
                        block_range=(b0, b1))
        shards.append((eng, e0, e1))
    p_sh = _dev(theta0, "f32")
    for s in range(1, 9):
        g = _dev(oracle.synth(42, s, 0, d, "f32"), "f32")
        full.step(p_full, g, 1e-2)
        for eng, e0, e1 in shards:
            eng.step(p_sh[e0:e1], g[e0:e1], 1e-2)
    torch.cuda.synchronize()
    assert torch.equal(p_full, p_sh)
    codes = np.concatenate([e.error_buffer().codes for e, _, _ in shards])
    assert np.array_equal(codes, full.error_buffer().codes)


def test_kernel_counts_and_library_is_native():
    """The step runs through libmicroadam_cuda.so (no fallback path exists)."""
    import paper_2405_15593_b200 as pkg
    d = 12 * 4096  # whole blocks: one fused launch per step (a partial tail adds one)
    eng = pkg.MicroAdam(d, dict(lr=1e-3))
    params = _dev(oracle.synth(1, 0, 0, d, "f32"), "f32")
    g = _dev(oracle.synth(42, 1, 0, d, "f32"), "f32")
    for _ in range(3):
        eng.step(params, g, 1e-3)
    eng.synchronize()
    assert eng.kernel_launches() == 3
    import os
    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert "libmicroadam_cuda.so" in maps


@pytest.mark.parametrize("kernel", sorted(KERNELS))
def test_persistent_spikes_duplicate_window_coordinates(kernel):
    # the same coordinates win every step: each window row repeats them, so
    # ADAM_STATS re-sums duplicated coordinates across all m rows.
    rng = np.random.default_rng(5)
    spikes = rng.choice(50_000, 400, replace=False)

    def g(s):
        x = oracle.synth(11, s, 0, 50_000) * 1e-3
        x[spikes] += 50.0 + s
        return x
    run_parity(50_000, dict(lr=1e-2, window=12), gdt="bf16", pdt="f32", vdt="bf16", steps=16,
               grad_fn=g, kernel=kernel)


@pytest.mark.parametrize("density,m", [(0.015, 10), (0.002, 30), (0.01, 127), (0.004, 256)])
def test_warp_kernel_shapes(density, m):
    run_parity(4096 * 9, dict(lr=1e-2, density=density, window=m), gdt="bf16", pdt="bf16",
               vdt="bf16", steps=min(m + 3, 20))


@pytest.mark.parametrize("bad", [np.inf, -np.inf, np.nan])
def test_nonfinite_flag_after_warm_threshold(bad):
    # the fast path (carried threshold) is active from step ~3: a non-finite
    # gradient there must still raise the flag (exact re-check on that path).
    from paper_2405_15593_b200 import InvalidArgument, MicroAdam
    d = 4096 * 6
    eng = MicroAdam(d, dict(lr=1e-2), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16",
                    finite_mode="flag")
    params = _dev(oracle.synth(1, 0, 0, d, "bf16"), "bf16")
    for s in range(1, 7):
        eng.step(params, _dev(oracle.synth(42, s, 0, d, "bf16"), "bf16"), 1e-2)
    eng.synchronize()
    g = oracle.synth(42, 7, 0, d, "bf16")
    g[4096 * 3 + 77] = bad
    eng.step(params, _dev(g, "bf16"), 1e-2)
    with pytest.raises(InvalidArgument):
        eng.synchronize()


@pytest.mark.parametrize("scale", [2.0 ** 120, 2.0 ** -130, 2.0 ** 300])
def test_fp64_magnitudes_outside_fp32_filter(scale):
    # |a| beyond the fp32 filter's safe range (or in fp32 denormals): the
    # kernel must fall back to the exact path and stay bit-exact.
    run_parity(4096 * 5, dict(lr=1e-3), gdt="f64", pdt="f64", vdt="f64", steps=6,
               grad_fn=lambda s: oracle.synth(7, s, 0, 4096 * 5) * scale)


def test_bf16_subnormal_window_values():
    # window values below 2^-126 round to bf16 subnormals (F2F.BF16.F64 on the
    # device vs the oracle's software RNE).
    run_parity(4096 * 3, dict(lr=1e-3), gdt="f64", pdt="f64", vdt="bf16", steps=5,
               grad_fn=lambda s: oracle.synth(5, s, 0, 4096 * 3) * 2.0 ** -133)


def test_reference_side_adapter_drives_reference_run_loop():
    """INTEGRATION.md's adapter, compiled against the unmodified reference
    headers/sources (oracle/_ref/adapter_check), run through the reference's
    own run() loop: every iterate bit-identical to the reference optimizer."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(oracle.__file__), "_ref", "adapter_check")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/adapter_check not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "adapter ok" in out.stdout


@pytest.mark.parametrize("bits,block,bucket", [(1, 4096, 64), (2, 4096, 64), (3, 1000, 8), (5, 4096, 128),
                                               (8, 512, 16), (12, 4096, 64), (16, 2048, 32), (24, 1000, 8),
                                               (23, 8192, 64)])
def test_other_code_widths_vs_unmodified_reference(bits, block, bucket):
    # QuantizedErrorBuffer with bits != 4 (quantize.cpp:102-128 LSB-first bit
    # stream, max_code = 2^bits - 1, bits up to the reference's 24): generic
    # kernel, fp64, bit-exact
    hp = dict(lr=1e-2, window=4, bits=bits, block=block, bucket=bucket)
    run_parity(20_011, hp, gdt="f64", pdt="f64", vdt="f64", steps=8,
               check_reference=oracle.reference_available())
