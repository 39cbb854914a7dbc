"""C ABI checks that need no GPU: the library loads, exports every symbol the
header declares, validates configs exactly where HyperParams::validate /
BlockLayout throw (optim.cpp:7-30, compress.cpp:19-33), derives the reference
layout, and refuses to run without a device (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

import oracle
from tests.conftest import ROOT, cuda_available

HEADER = os.path.join(ROOT, "include", "microadam_cuda.h")


@pytest.fixture(scope="module")
def ma():
    import paper_2405_15593_b200 as pkg
    if not os.path.exists(pkg.LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", ROOT, "lib"])
    return pkg


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"MA_API\s+[\w\s\*]+?\b(ma_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol(ma):
    syms = declared_symbols()
    assert len(syms) >= 19
    L = ma.lib()
    for s in syms:
        assert hasattr(L, s), s
    out = subprocess.check_output(["nm", "-D", "--defined-only", ma.LIB_PATH], text=True)
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(syms) <= exported
    assert set(syms) == set(ma._capi.EXPORTED)


def test_header_is_plain_c():
    for std in ("-std=c99", "-std=c11"):
        subprocess.check_call(["gcc", std, "-Wall", "-Werror", "-fsyntax-only", "-x", "c", HEADER])
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-x", "c",
                           os.path.join(ROOT, "include", "ma_synth.h")])


def test_cpp_host_api_links(ma, tmp_path):
    """A reference-style C++ caller compiles and links against the library."""
    src = tmp_path / "caller.cpp"
    src.write_text(
        '#include "paper_2405_15593_b200/csrc/microadam_b200.hpp"\n'
        "int main(int argc, char**) {\n"
        "  microadam_b200::HyperParams hp; hp.validate();\n"
        "  if (argc > 5) {  // link check only: never runs without a GPU\n"
        "    microadam_b200::MicroAdamOptimizer opt(microadam_b200::Vec(8, 0.0), hp);\n"
        "    microadam_b200::Optimizer& o = opt; o.step(microadam_b200::Vec(8, 1.0));\n"
        "    microadam_b200::MicroAdam eng(8, hp);\n"
        "    std::vector<const void*> srcs(2, nullptr);\n"
        "    eng.step_reduce(nullptr, nullptr, srcs, 0.5f, 1e-3);\n"
        "  }\n"
        "  return hp.resolve_k(1000) == 10 ? 0 : 1;\n}\n")
    exe = tmp_path / "caller"
    libdir = os.path.dirname(ma.LIB_PATH)
    subprocess.check_call(["g++", "-std=c++17", "-Wall", "-Werror", f"-I{ROOT}", str(src), "-o",
                           str(exe), f"-L{libdir}", "-lmicroadam_cuda", f"-Wl,-rpath,{libdir}"])
    subprocess.check_call([str(exe)])


def _cfg(ma, **kw):
    cfg = ma._capi.default_config()
    for k, v in kw.items():
        if hasattr(cfg.hp, k):
            setattr(cfg.hp, k, v)
        else:
            setattr(cfg, k, v)
    return cfg


def _validate(ma, dim=1000, **kw):
    return ma.lib().ma_validate(C.byref(_cfg(ma, **kw)), dim)


def test_defaults_mirror_reference(ma):  # optim.hpp:15-30, test_optim.cpp:46-56
    cfg = ma._capi.default_config()
    hp = cfg.hp
    assert (hp.beta1, hp.beta2, hp.eps, hp.window, hp.density, hp.bits, hp.block, hp.bucket) == (
        0.9, 0.999, 1e-8, 10, 0.01, 4, 4096, 64)
    assert ma.HyperParams().resolve_k(1000) == 10
    assert ma.HyperParams().resolve_k(50) == 1
    assert ma.HyperParams(k=7).resolve_k(1000) == 7
    with pytest.raises(ValueError):
        ma.HyperParams(k=7).resolve_k(5)


@pytest.mark.parametrize("field,value", [
    ("beta1", 1.0), ("beta1", 0.0), ("beta2", 1.0), ("eps", 0.0), ("lr", 0.0),
    ("weight_decay", -1.0), ("window", 0), ("density", 0.0), ("density", 1.5), ("bits", 25),
    ("bits", 0), ("block", 40000), ("block", 0), ("bucket", 0),
])
def test_invalid_hyperparams_rejected(ma, field, value):  # optim.cpp:7-21
    assert _validate(ma, **{field: value}) == ma._capi.MA_ERR_INVALID_ARG
    with pytest.raises(ValueError):
        ma.HyperParams(**{field: value}).validate()


def test_empty_vector_rejected(ma):  # optim.cpp:136 "empty parameter vector"
    assert _validate(ma, dim=0) == ma._capi.MA_ERR_INVALID_ARG
    assert _validate(ma, dim=1) == ma._capi.MA_OK


def test_k_exceeding_dim_rejected(ma):  # optim.cpp:23-26
    assert _validate(ma, dim=5, k=7) == ma._capi.MA_ERR_INVALID_ARG


@pytest.mark.parametrize("kw", [dict(block=16384, bits=3), dict(window=1025),
                                dict(window=300, blockwise=0),
                                dict(bucket=100, bits=3), dict(bucket=100, lossless_error=1)])
def test_unsupported_device_shapes_are_explicit(ma, kw):
    assert _validate(ma, dim=100_000, **kw) == ma._capi.MA_ERR_UNSUPPORTED


def test_big_blocks(ma):
    # BlockLayout allows B_d up to 32767 (compress.hpp:23): the big-block kernel
    assert _validate(ma, dim=100_000, block=16384) == ma._capi.MA_OK
    assert _validate(ma, dim=100_000, block=32767) == ma._capi.MA_OK
    # beyond the reference's limit: its BlockLayout throws (std::invalid_argument)
    assert _validate(ma, dim=100_000, block=40000) == ma._capi.MA_ERR_INVALID_ARG


def test_long_windows(ma):
    # HyperParams::validate only needs window >= 1 (optim.cpp:13): m up to 1024 on device
    assert _validate(ma, dim=100_000, window=300) == ma._capi.MA_OK
    assert _validate(ma, dim=100_000, window=1024) == ma._capi.MA_OK


@pytest.mark.parametrize("kw", [dict(bucket=100), dict(block=4095), dict(bucket=100_000),
                                dict(block=1001, bucket=7)])
def test_buckets_straddling_blocks_are_supported(ma, kw):
    # quantize.cpp:142-162 buckets the whole vector: B_q need not divide B_d
    # (the paper's B_q = 100,000): per-bucket re-quantization kernel
    assert _validate(ma, dim=300_000, **kw) == ma._capi.MA_OK


def test_single_block_allows_any_bucket(ma):
    # buckets may straddle nothing when one block spans d (block = min(block, d))
    assert _validate(ma, dim=3000, bucket=100) == ma._capi.MA_OK
    assert _validate(ma, dim=37, block=37, bucket=5) == ma._capi.MA_OK


# SURVEY.md §8 size table (B_d=4096, B_q=64, 1%).
@pytest.mark.parametrize("dim,blocks,row_width,buckets,code_bytes", [
    (1_000_000, 245, 10_045, 15_625, 500_000),
    (110_000_000, 26_856, 1_101_096, 1_718_750, 55_000_000),
    (1_300_000_000, 317_383, 13_012_703, 20_312_500, 650_000_000),
    (6_738_415_616, 1_645_121, 67_449_961, 105_287_744, 3_369_207_808),
])
def test_layout_matches_survey_table(ma, dim, blocks, row_width, buckets, code_bytes):
    lay = ma.layout(dim)
    assert (lay.num_blocks, lay.row_width, lay.num_buckets, lay.code_bytes) == (
        blocks, row_width, buckets, code_bytes)
    assert lay.per_block_k == 41


@pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")
def test_per_block_k_matches_reference_from_density(ma):  # compress.cpp:28-33
    L = oracle.ref_lib()
    for block in (1, 7, 64, 1000, 4096, 8192):
        for density in (0.001, 0.01, 0.0123, 0.05, 0.25, 1.0):
            lay = ma.layout(block, dict(block=block, density=density, bucket=1))
            assert lay.per_block_k == L.ref_per_block_k(block, block, density)


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_device(ma):
    with pytest.raises(ma.MicroAdamError) as e:
        ma.MicroAdam(1000, dict())
    assert e.value.status == ma._capi.MA_ERR_CUDA
    assert "no CPU fallback" in str(e.value)


def test_oracle_not_imported_by_product():
    pkg_dir = os.path.join(ROOT, "paper_2405_15593_b200")
    for dirpath, _, files in os.walk(pkg_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".hpp", ".cuh")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text and "libmicroadam_ref" not in text, f


def test_global_mode_shapes(ma):
    # blockwise = false (the reference default) runs on device for any d
    # (int64 window indices) with bucket | 4096 (ma_global.cu); d <= 8192 stays
    # a single block
    assert _validate(ma, dim=100_000, blockwise=0) == ma._capi.MA_OK
    assert _validate(ma, dim=5_000, blockwise=0, bucket=100) == ma._capi.MA_OK
    assert _validate(ma, dim=100_000, blockwise=0, bucket=100) == ma._capi.MA_ERR_UNSUPPORTED
    assert _validate(ma, dim=3_000_000_000, blockwise=0) == ma._capi.MA_OK
    assert _validate(ma, dim=13_015_864_320, blockwise=0) == ma._capi.MA_OK


def test_lossless_blockwise_is_supported(ma):
    # MicroAdamOptimizer(..., lossless_error = true) (optim.hpp:103-104): dense fp64 EF
    assert _validate(ma, dim=100_000, lossless_error=1) == ma._capi.MA_OK
    assert _validate(ma, dim=100_000, lossless_error=1, blockwise=0) == ma._capi.MA_OK


def test_code_widths(ma):
    assert _validate(ma, dim=100_000, bits=3, block=1000, bucket=8) == ma._capi.MA_OK
    assert _validate(ma, dim=100_000, bits=3, block=1001, bucket=7) == ma._capi.MA_ERR_UNSUPPORTED
    assert _validate(ma, dim=100_000, bits=12) == ma._capi.MA_OK      # up to the reference's 24
    assert _validate(ma, dim=100_000, bits=24, block=1000, bucket=8) == ma._capi.MA_OK
    assert _validate(ma, dim=100_000, bits=12, block=1001, bucket=7) == ma._capi.MA_ERR_UNSUPPORTED
    assert _validate(ma, dim=100_000, bits=2, blockwise=0) == ma._capi.MA_ERR_UNSUPPORTED
