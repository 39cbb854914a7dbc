"""Global Top-K mode on the device for d > 8192 (SURVEY.md §8 a16 / §8(f)
rank 4; the reference's default MicroAdamOptimizer(blockwise=false),
topk_global compress.cpp:66-71).

fp64 θ/g/window: bit-exact against the UNMODIFIED reference every step (θ, EF
codes, bucket (lo, hi), window row). bf16/f32 dtypes: bit-exact against the
composed oracle (block = d). Ties at the k-th key (16-level gradients) take
the lowest indices; checkpoints are byte-identical to the reference's; the
host drop-in class matches the reference's StepReport.
"""
import numpy as np
import pytest

import oracle
from tests.conftest import cuda_available
from tests.test_gpu_parity import _bits, _dev, _host, _torch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]
needs_ref = pytest.mark.skipif(not oracle.reference_available(), reason="needs /root/reference")


def _global_engine(d, hp, dt, vdt, cand_cap=None):
    import os
    from paper_2405_15593_b200 import MicroAdam
    if cand_cap is not None:
        os.environ["MA_GLOBAL_CAND_CAP"] = str(cand_cap)
    try:
        return MicroAdam(d, hp, param_dtype=dt, grad_dtype=dt, value_dtype=vdt, blockwise=False)
    finally:
        os.environ.pop("MA_GLOBAL_CAND_CAP", None)


@needs_ref
@pytest.mark.parametrize("d,hp,levels", [
    (50_000, dict(lr=1e-2, window=4), False),
    (100_003, dict(lr=1e-2, window=3, bucket=32), False),
    (40_000, dict(lr=1e-2, window=5, k=777), True),   # 16-level grads: ties at K*
])
def test_global_fp64_matches_unmodified_reference(d, hp, levels):
    torch = _torch()
    th0 = oracle.synth(1, 0, 0, d)
    ref = oracle.Reference(th0, hp, blockwise=False)
    eng = _global_engine(d, hp, "f64", "f64")
    p = _dev(th0, "f64")
    for s in range(1, 8):
        g = oracle.synth(42, s, 0, d, levels=levels)
        ref.step(g)
        eng.step(p, _dev(g, "f64"), hp["lr"])
        torch.cuda.synchronize()
        st = ref.state()
        head = eng.counters()[1]
        slot = (head + hp["window"] - 1) % hp["window"]
        assert np.array_equal(eng.window().indices[slot], st.last_idx), f"selection @ {s}"
        assert np.array_equal(eng.error_buffer().codes, st.codes), f"codes @ {s}"
        assert np.array_equal(_bits(eng.error_buffer().lo), _bits(st.lo)), f"lo @ {s}"
        assert np.array_equal(_bits(_host(p)), _bits(st.params)), f"θ @ {s}"


@pytest.mark.parametrize("dt,cap", [("bf16", None), ("f32", None), ("bf16", 0), ("f32", 3)])
def test_global_low_precision_matches_composed_oracle(dt, cap):
    # cap: capacity of the candidate-key buffer of the radix select's last
    # three digits; 0 / 3 force the overflow path (full passes)
    d = 30_011
    hp = dict(lr=1e-2, window=4, density=0.02)
    torch = _torch()
    th0 = _host(_dev(oracle.synth(1, 0, 0, d, dt), dt))
    orc = oracle.Oracle(th0, dict(hp, block=d), param_dtype=dt, value_dtype="bf16")
    eng = _global_engine(d, hp, dt, "bf16", cand_cap=cap)
    p = _dev(th0, dt)
    for s in range(1, 8):
        g = _host(_dev(oracle.synth(42, s, 0, d, dt), dt))
        orc.step(g, hp["lr"])
        eng.step(p, _dev(g, dt), hp["lr"])
        torch.cuda.synchronize()
        so = orc.state()
        assert np.array_equal(eng.error_buffer().codes, so.codes), f"codes @ {s}"
        assert np.array_equal(_bits(_host(p)), _bits(so.params)), f"θ @ {s}"
        w = eng.window()
        for r in range(eng.counters()[2]):
            assert np.array_equal(w.indices[r], so.win_idx[r])
            assert np.array_equal(_bits(w.values[r]), _bits(so.win_val[r]))


@needs_ref
def test_global_dropin_class_and_checkpoint_match_reference(tmp_path):
    from paper_2405_15593_b200 import MicroAdamOptimizer
    d, hp = 20_000, dict(lr=1e-2, window=3)
    th0 = oracle.synth(1, 0, 0, d)
    opt = MicroAdamOptimizer(th0, hp, blockwise=False)
    ref = oracle.Reference(th0, hp, blockwise=False)
    for s in range(1, 6):
        g = oracle.synth(42, s, 0, d)
        rep = opt.step(g)
        rrep = ref.step(g)
        assert np.array_equal(_bits(opt.params()), _bits(ref.state().params))
        assert rep.update_nnz == rrep["update_nnz"]
        assert abs(rep.grad_norm - rrep["grad_norm"]) <= 1e-12 * rrep["grad_norm"]
        assert abs(rep.error_norm - rrep["error_norm"]) <= 1e-12 * max(rrep["error_norm"], 1e-300)
    a, b = str(tmp_path / "ref.madm"), str(tmp_path / "dev.madm")
    ref.save_checkpoint(a)
    eng = _global_engine(d, hp, "f64", "f64")
    p = _dev(th0, "f64")
    for s in range(1, 6):
        eng.step(p, _dev(oracle.synth(42, s, 0, d), "f64"), hp["lr"])
    eng.synchronize()
    eng.save_checkpoint(b, p)
    assert open(a, "rb").read() == open(b, "rb").read()


def test_global_mode_tie_heavy_f32():
    # 16-level gradients (ties at the k-th key), m = 2, f32 window values
    hp = dict(lr=1e-2, window=2, density=0.003)
    d = 12_345
    torch = _torch()
    th0 = _host(_dev(oracle.synth(1, 0, 0, d, "f32"), "f32"))
    orc = oracle.Oracle(th0, dict(hp, block=d), param_dtype="f32", value_dtype="f32")
    eng = _global_engine(d, hp, "f32", "f32", cand_cap=5)  # ties overflow the candidate buffer
    p = _dev(th0, "f32")
    for s in range(1, 6):
        g = _host(_dev(oracle.synth(5, s, 0, d, "f32", levels=True), "f32"))
        orc.step(g, hp["lr"])
        eng.step(p, _dev(g, "f32"), hp["lr"])
    torch.cuda.synchronize()
    so = orc.state()
    assert np.array_equal(_bits(_host(p)), _bits(so.params))
    assert np.array_equal(eng.error_buffer().codes, so.codes)


@pytest.mark.parametrize("dt,density", [("bf16", 0.03), ("f32", 0.08), ("bf16", 0.08)])
def test_global_dense_window_chunks(dt, density):
    # m = 8: ~980 (3%) or ~2600 (8%) window entries per 4096-chunk; the latter
    # exceed the staged ADAM_STATS path (2048) and take the dense one
    hp = dict(lr=1e-2, window=8, density=density)
    d = 32_001  # the oracle's block limit (block = d in global mode)
    th0 = _host(_dev(oracle.synth(1, 0, 0, d, dt), dt))
    orc = oracle.Oracle(th0, dict(hp, block=d), param_dtype=dt, value_dtype="bf16")
    eng = _global_engine(d, hp, dt, "bf16")
    p = _dev(th0, dt)
    torch = _torch()
    for s in range(1, 11):
        g = _host(_dev(oracle.synth(42, s, 0, d, dt), dt))
        orc.step(g, hp["lr"])
        eng.step(p, _dev(g, dt), hp["lr"])
        torch.cuda.synchronize()
        assert np.array_equal(_bits(_host(p)), _bits(orc.state().params)), f"θ @ {s}"
    assert np.array_equal(eng.error_buffer().codes, orc.state().codes)


@pytest.mark.parametrize("dt,levels", [("bf16", False), ("f32", True)])
def test_global_carried_bracket_scale_jumps(dt, levels):
    # The select carries a bracket around the previous step's K* (g_bracket):
    # gradient scale jumps of 2^±12 move K* far outside it (fallback to the
    # full digit passes, then a re-centred bracket), steady steps keep K*
    # inside; 16-level gradients put many ties at K* inside the bracket.
    d = 32_003  # the composed oracle takes the whole vector as one block (<= 32767)
    hp = dict(lr=1e-2, window=4, density=0.01)
    scales = [1.0, 1.0, 1.0, 2.0 ** 12, 2.0 ** 12, 2.0 ** 12, 2.0 ** -12, 1.0, 1.0, 1.0, 1.0]
    torch = _torch()
    th0 = _host(_dev(oracle.synth(1, 0, 0, d, dt), dt))
    orc = oracle.Oracle(th0, dict(hp, block=d), param_dtype=dt, value_dtype="bf16")
    eng = _global_engine(d, hp, dt, "bf16")
    p = _dev(th0, dt)
    for s, sc in enumerate(scales, start=1):
        g = _host(_dev(oracle.synth(42, s, 0, d, dt, levels=levels) * sc, dt))
        orc.step(g, hp["lr"])
        eng.step(p, _dev(g, dt), hp["lr"])
        torch.cuda.synchronize()
        so = orc.state()
        w = eng.window()
        slot = (eng.counters()[1] + hp["window"] - 1) % hp["window"]
        assert np.array_equal(w.indices[slot], so.win_idx[slot]), f"selection @ {s}"
        assert np.array_equal(eng.error_buffer().codes, so.codes), f"codes @ {s}"
        assert np.array_equal(_bits(_host(p)), _bits(so.params)), f"θ @ {s}"


def test_global_tiled_allocation_scan(monkeypatch):
    # the three-launch chunk allocation (g_alloc_tiles / g_alloc_scan /
    # g_alloc_final) that large vectors use, forced at a size the composed
    # oracle checks; 16-level gradients put ties at K* across chunks
    monkeypatch.setenv("MA_GLOBAL_ALLOC_TILED", "1")
    d = 31_000
    hp = dict(lr=1e-2, window=3, density=0.05)
    torch = _torch()
    th0 = _host(_dev(oracle.synth(1, 0, 0, d, "bf16"), "bf16"))
    orc = oracle.Oracle(th0, dict(hp, block=d), param_dtype="bf16", value_dtype="bf16")
    eng = _global_engine(d, hp, "bf16", "bf16")
    p = _dev(th0, "bf16")
    for s in range(1, 7):
        g = _host(_dev(oracle.synth(9, s, 0, d, "bf16", levels=s % 2 == 0), "bf16"))
        orc.step(g, hp["lr"])
        eng.step(p, _dev(g, "bf16"), hp["lr"])
        torch.cuda.synchronize()
        so = orc.state()
        slot = (eng.counters()[1] + hp["window"] - 1) % hp["window"]
        assert np.array_equal(eng.window().indices[slot], so.win_idx[slot]), f"selection @ {s}"
        assert np.array_equal(_bits(_host(p)), _bits(so.params)), f"θ @ {s}"


@pytest.mark.parametrize("bucket,levels", [(8, False), (16, True), (64, True), (256, False)])
def test_global_fp32_requant_buckets(bucket, levels):
    # g_requant8f (bf16 gradients, whole chunks) for every register bucket
    # width (B_q = 8 .. 256: 1 .. 32 threads per bucket), tie-heavy gradients
    # (constant / two-valued buckets send whole buckets to the fp64 path);
    # d leaves a partial last chunk for the fp64 kernel
    d = 4096 * 6 + 1000
    hp = dict(lr=1e-2, window=3, density=0.02, bucket=bucket)
    torch = _torch()
    th0 = _host(_dev(oracle.synth(1, 0, 0, d, "bf16"), "bf16"))
    orc = oracle.Oracle(th0, dict(hp, block=d), param_dtype="bf16", value_dtype="bf16")
    eng = _global_engine(d, hp, "bf16", "bf16")
    p = _dev(th0, "bf16")
    for s in range(1, 7):
        g = _host(_dev(oracle.synth(11, s, 0, d, "bf16", levels=levels) * (2.0 ** (3 * (s % 3))), "bf16"))
        orc.step(g, hp["lr"])
        eng.step(p, _dev(g, "bf16"), hp["lr"])
        torch.cuda.synchronize()
        so = orc.state()
        eb = eng.error_buffer()
        assert np.array_equal(eb.codes, so.codes), f"codes @ {s}"
        assert np.array_equal(_bits(eb.lo), _bits(so.lo)), f"lo @ {s}"
        assert np.array_equal(_bits(eb.hi), _bits(so.hi)), f"hi @ {s}"
        assert np.array_equal(_bits(_host(p)), _bits(so.params)), f"θ @ {s}"
