"""Lossless error feedback on the device: MicroAdamOptimizer(theta0, hp,
blockwise, lossless_error = true) (optim.hpp:103-104, optim.cpp:172-173) keeps
the residual dense in fp64. Bit-exact against the UNMODIFIED reference (θ,
window rows, error vector, StepReport), the reference's conservation test
(test_optim.cpp:204-219: e_new + embed(selection) == a, bitwise), the
error_buffer() logic error, and byte-identical MADM checkpoints (lossless flag
set, dense error stored).
"""
import numpy as np
import pytest

import oracle
from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not oracle.reference_available(), reason="needs /root/reference")]


def _bits(x):
    return np.asarray(x, np.float64).view(np.uint64)


@pytest.mark.parametrize("d,hp,blockwise", [(30_011, dict(lr=1e-2, window=4), True),
                                            (4096 * 3, dict(lr=1e-2, window=3, block=1024, density=0.02), True),
                                            (30_011, dict(lr=1e-2, window=4), False),   # global Top-K (ma_global.cu)
                                            (50_000, dict(lr=1e-2, window=3, k=333), False)])
def test_lossless_matches_reference_and_conserves(d, hp, blockwise):
    from paper_2405_15593_b200 import MicroAdamOptimizer
    th0 = oracle.synth(1, 0, 0, d)
    opt = MicroAdamOptimizer(th0, hp, blockwise=blockwise, lossless_error=True)
    ref = oracle.Reference(th0, hp, blockwise=blockwise, lossless=True)
    assert opt.lossless()
    e_prev = np.zeros(d)
    for s in range(1, 8):
        g = oracle.synth(42, s, 0, d)
        a = g + e_prev                     # optim.cpp:166-168 (fp64, same rounding)
        rep = opt.step(g)
        rrep = ref.step(g)
        st = ref.state()
        assert np.array_equal(_bits(opt.params()), _bits(st.params)), f"θ @ {s}"
        assert np.array_equal(opt.last_selection().indices, st.last_idx)
        e_new = opt.error_vector()
        assert np.array_equal(_bits(e_new), _bits(ref.error_vector())), f"error @ {s}"
        emb = e_new.copy()                 # conservation: e_new + embed(sel) == a
        emb[opt.last_selection().indices] = opt.last_selection().values
        assert np.array_equal(_bits(emb), _bits(a)), f"conservation @ {s}"
        assert rep.update_nnz == rrep["update_nnz"]
        assert abs(rep.error_norm - rrep["error_norm"]) <= 1e-12 * max(rrep["error_norm"], 1e-300)
        e_prev = e_new
    with pytest.raises(RuntimeError, match="dense error storage"):
        opt.error_buffer()


def test_lossless_checkpoint_bytes_equal_reference(tmp_path):
    from paper_2405_15593_b200 import MicroAdamOptimizer
    d, hp = 20_000, dict(lr=1e-2, window=3)
    th0 = oracle.synth(1, 0, 0, d)
    ref = oracle.Reference(th0, hp, lossless=True)
    opt = MicroAdamOptimizer(th0, hp, blockwise=True, lossless_error=True)
    for s in range(1, 6):
        g = oracle.synth(42, s, 0, d)
        ref.step(g)
        opt.step(g)
    a, b = str(tmp_path / "ref.madm"), str(tmp_path / "dev.madm")
    ref.save_checkpoint(a)
    opt.save_checkpoint(b)
    assert open(a, "rb").read() == open(b, "rb").read()
    resumed = MicroAdamOptimizer(np.zeros(d), hp, blockwise=True, lossless_error=True)
    resumed.load_checkpoint(b)
    for s in range(6, 9):
        g = oracle.synth(42, s, 0, d)
        ref.step(g)
        resumed.step(g)
    assert np.array_equal(_bits(resumed.params()), _bits(ref.state().params))
    assert np.array_equal(_bits(resumed.error_vector()), _bits(ref.error_vector()))
