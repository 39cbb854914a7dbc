"""MADM v1 checkpoints (checkpoint.hpp:28-33,
checkpoint.cpp:50-140).

CPU part: the reference's own save/load round trip through the shim (pins
the format the device writer must reproduce). GPU part (-m gpu): the device
writer produces byte-identical files to the reference's save_checkpoint in
fp64 mode, its files load in the reference loader in every dtype, a device
handle resumes bit-exactly from its own and from the reference's
checkpoints, and malformed files are rejected like the reference does
(test_checkpoint.cpp:49-84 is the reference's round-trip test).
"""
import numpy as np
import pytest

import oracle
from tests.conftest import cuda_available

needs_ref = pytest.mark.skipif(not oracle.reference_available(), reason="needs /root/reference")


@needs_ref
def test_reference_round_trip(tmp_path):  # test_checkpoint.cpp:49-84
    d, hp = 3001, dict(lr=1e-2, window=3, bucket=16, block=512)
    ref = oracle.Reference(oracle.synth(1, 0, 0, d), hp)
    for s in range(1, 6):
        ref.step(oracle.synth(42, s, 0, d))
    path = str(tmp_path / "ref.madm")
    ref.save_checkpoint(path)
    head, theta = oracle.ref_load_checkpoint(path, d)
    st = ref.state()
    assert head == dict(dim=d, step=5, capacity=3, row_width=ref.row_width, head=5 % 3, filled=3)
    assert np.array_equal(theta.view(np.uint64), st.params.view(np.uint64))
    raw = open(path, "rb").read()
    assert raw[:5] == b"MADM\x01"
    with open(path, "wb") as f:
        f.write(b"MADX" + raw[4:])
    with pytest.raises(ValueError, match="bad magic"):
        oracle.ref_load_checkpoint(path, d)


def _bits(x):
    return np.asarray(x, np.float64).view(np.uint64)


def _torch_dt(dt):
    import torch
    return {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dt]


def _dev(x, dt):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float64)).to(_torch_dt(dt)).cuda()


def _engine(d, hp, dt):
    from paper_2405_15593_b200 import MicroAdam
    vdt = "f64" if dt == "f64" else "bf16"
    return MicroAdam(d, hp, param_dtype=dt, grad_dtype=dt, value_dtype=vdt)


def _same_state(a, pa, b, pb):
    import torch
    assert torch.equal(pa, pb)
    assert a.counters()[:3] == b.counters()[:3]
    assert np.array_equal(a.counters()[3], b.counters()[3])
    ea, eb = a.error_buffer(), b.error_buffer()
    assert np.array_equal(ea.codes, eb.codes)
    assert np.array_equal(_bits(ea.lo), _bits(eb.lo)) and np.array_equal(_bits(ea.hi), _bits(eb.hi))
    wa, wb = a.window(), b.window()
    assert np.array_equal(wa.indices, wb.indices)
    assert np.array_equal(_bits(wa.values), _bits(wb.values))


@pytest.mark.parametrize("d", [50_003, 4096 * 5])
@needs_ref
@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
def test_device_checkpoint_bytes_equal_reference(tmp_path, d):
    hp = dict(lr=1e-2, window=4)
    th0 = oracle.synth(1, 0, 0, d)
    ref = oracle.Reference(th0, hp)
    eng = _engine(d, hp, "f64")
    p = _dev(th0, "f64")
    for s in range(1, 8):
        g = oracle.synth(42, s, 0, d)
        ref.step(g)
        eng.step(p, _dev(g, "f64"), 1e-2)
    eng.synchronize()
    a, b = str(tmp_path / "ref.madm"), str(tmp_path / "dev.madm")
    ref.save_checkpoint(a)
    eng.save_checkpoint(b, p)
    assert open(a, "rb").read() == open(b, "rb").read()


@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
def test_device_checkpoint_loads_in_reference_and_resumes(tmp_path, dt):
    d, hp = 4096 * 6 + 100, dict(lr=1e-2, window=5)
    th0 = oracle.synth(1, 0, 0, d, dt)
    full, pf = _engine(d, hp, dt), _dev(th0, dt)
    part, pp = _engine(d, hp, dt), _dev(th0, dt)
    grads = [_dev(oracle.synth(42, s, 0, d, dt), dt) for s in range(1, 11)]
    for g in grads:
        full.step(pf, g, 1e-2)
    for g in grads[:6]:
        part.step(pp, g, 1e-2)
    part.synchronize()
    path = str(tmp_path / "part.madm")
    part.save_checkpoint(path, pp)
    if oracle.reference_available():
        head, theta = oracle.ref_load_checkpoint(path, d)
        assert head["dim"] == d and head["step"] == 6 and head["filled"] == 5
        assert np.array_equal(_bits(theta), _bits(pp.double().cpu().numpy()))
    resumed, pr = _engine(d, hp, dt), _dev(np.zeros(d), dt)
    resumed.load_checkpoint(path, pr)
    for g in grads[6:]:
        resumed.step(pr, g, 1e-2)
    resumed.synchronize()
    full.synchronize()
    _same_state(full, pf, resumed, pr)


@needs_ref
@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
def test_device_resumes_from_reference_checkpoint(tmp_path):
    d, hp = 20_001, dict(lr=1e-2, window=3)
    th0 = oracle.synth(1, 0, 0, d)
    ref = oracle.Reference(th0, hp)
    for s in range(1, 6):
        ref.step(oracle.synth(42, s, 0, d))
    path = str(tmp_path / "ref.madm")
    ref.save_checkpoint(path)
    eng, p = _engine(d, hp, "f64"), _dev(np.zeros(d), "f64")
    eng.load_checkpoint(path, p)
    for s in range(6, 10):
        g = oracle.synth(42, s, 0, d)
        ref.step(g)
        eng.step(p, _dev(g, "f64"), 1e-2)
    eng.synchronize()
    st = ref.state()
    assert np.array_equal(_bits(p.cpu().numpy()), _bits(st.params))
    assert np.array_equal(eng.error_buffer().codes, st.codes)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
def test_malformed_checkpoints_rejected(tmp_path):
    from paper_2405_15593_b200 import InvalidArgument
    from paper_2405_15593_b200._capi import MicroAdamError
    d, hp = 8192, dict(lr=1e-2, window=2)
    eng, p = _engine(d, hp, "f32"), _dev(oracle.synth(1, 0, 0, d, "f32"), "f32")
    eng.step(p, _dev(oracle.synth(42, 1, 0, d, "f32"), "f32"), 1e-2)
    path = str(tmp_path / "x.madm")
    eng.save_checkpoint(path, p)
    raw = open(path, "rb").read()
    for bad, what in ((b"MADX" + raw[4:], "bad magic"), (raw[:4] + b"\x02" + raw[5:], "version"),
                      (raw[:100], "truncated")):
        with open(path, "wb") as f:
            f.write(bad)
        with pytest.raises((InvalidArgument, MicroAdamError), match=what):
            eng.load_checkpoint(path, p)
    other = _engine(d + 4096, hp, "f32")
    with open(path, "wb") as f:
        f.write(raw)
    with pytest.raises((InvalidArgument, MicroAdamError), match="dimension"):
        other.load_checkpoint(path)
