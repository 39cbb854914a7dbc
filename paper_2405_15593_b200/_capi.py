"""ctypes binding of the C ABI in include/microadam_cuda.h (libmicroadam_cuda.so).

The library is built in-tree (``make lib`` / ``__graft_entry__.build()``) into
paper_2405_15593_b200/lib/. There is no fallback: if the library is missing or
no CUDA device is visible, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MA_LIB_PATH") or os.path.join(HERE, "lib", "libmicroadam_cuda.so")

# ma_status
MA_OK, MA_ERR_INVALID_ARG, MA_ERR_DIM, MA_ERR_NONFINITE, MA_ERR_CUDA, MA_ERR_NCCL, \
    MA_ERR_UNSUPPORTED, MA_ERR_STATE = range(8)
# ma_dtype
MA_F64, MA_F32, MA_BF16 = 0, 1, 2
DTYPE_CODES = {"f64": MA_F64, "f32": MA_F32, "bf16": MA_BF16}
# ma_finite_mode
MA_FINITE_FLAG, MA_FINITE_STRICT, MA_FINITE_OFF = 0, 1, 2

EXPORTED = [
    "ma_config_default", "ma_validate", "ma_layout", "ma_create", "ma_create_shard", "ma_destroy",
    "ma_step", "ma_step_host", "ma_sync", "ma_get_counters", "ma_read_error_buffer",
    "ma_read_window_row", "ma_write_state", "ma_set_params", "ma_get_layout",
    "ma_kernel_launches", "ma_last_error", "ma_version", "ma_fill_synthetic", "ma_debug_counters",
    "ma_save_checkpoint", "ma_load_checkpoint", "ma_step_front", "ma_scatter_rows", "ma_step_stats",
    "ma_read_error_vector", "ma_step_reduce", "ma_read_error_buffer_blocks", "ma_read_window_blocks",
    "ma_comm_unique_id", "ma_comm_init", "ma_comm_wrap", "ma_comm_destroy", "ma_comm_info",
    "ma_step_allgather", "ma_allgather_params", "ma_exchange_rows",
]


class Hyper(C.Structure):
    _fields_ = [
        ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double), ("lr", C.c_double),
        ("weight_decay", C.c_double), ("window", C.c_int64), ("density", C.c_double),
        ("k", C.c_int64), ("bits", C.c_int32), ("reserved0", C.c_int32), ("block", C.c_int64),
        ("bucket", C.c_int64),
    ]


class Config(C.Structure):
    _fields_ = [
        ("hp", Hyper), ("blockwise", C.c_int32), ("lossless_error", C.c_int32),
        ("param_dtype", C.c_int32), ("grad_dtype", C.c_int32), ("value_dtype", C.c_int32),
        ("finite_mode", C.c_int32),
    ]


class Report(C.Structure):
    _fields_ = [
        ("grad_norm", C.c_double), ("error_norm", C.c_double), ("empirical_q", C.c_double),
        ("update_nnz", C.c_int64), ("loss", C.c_double),
    ]


class Layout(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "dim", "block", "per_block_k", "num_blocks", "row_width", "num_buckets", "code_bytes",
        "kb_stride", "state_bytes")]


class MicroAdamError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


_lib = None


def lib():
    """Load libmicroadam_cuda.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
            "the MicroAdam device path has no CPU fallback")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    L.ma_config_default.argtypes = [P(Config)]
    L.ma_config_default.restype = None
    L.ma_validate.argtypes = [P(Config), C.c_int64]
    L.ma_layout.argtypes = [P(Config), C.c_int64, C.c_int64, C.c_int64, P(Layout)]
    L.ma_create.argtypes = [P(Config), C.c_int64, C.c_int, P(vp)]
    L.ma_create_shard.argtypes = [P(Config), C.c_int64, C.c_int64, C.c_int64, C.c_int, P(vp)]
    L.ma_destroy.argtypes = [vp]
    L.ma_step.argtypes = [vp, vp, vp, C.c_double, vp, P(Report)]
    L.ma_step_host.argtypes = [vp, vp, vp, C.c_double, P(Report)]
    L.ma_step_reduce.argtypes = [vp, vp, vp, P(vp), C.c_int32, C.c_float, C.c_double, vp, P(Report)]
    L.ma_sync.argtypes = [vp]
    L.ma_comm_unique_id.argtypes = [vp]
    L.ma_comm_init.argtypes = [vp, C.c_int32, C.c_int32, C.c_int, P(vp)]
    L.ma_comm_wrap.argtypes = [vp, P(vp)]
    L.ma_comm_destroy.argtypes = [vp]
    L.ma_comm_info.argtypes = [vp, P(C.c_int32), P(C.c_int32)]
    L.ma_step_allgather.argtypes = [vp, vp, C.c_int64, vp, C.c_double, vp, vp, P(Report)]
    L.ma_allgather_params.argtypes = [vp, vp, C.c_int64, vp, vp]
    L.ma_exchange_rows.argtypes = [vp, vp, vp, C.c_int64, vp, vp, vp, vp]
    L.ma_get_counters.argtypes = [vp, P(C.c_int64), P(C.c_int64), P(C.c_int64), P(C.c_int64)]
    L.ma_read_error_buffer.argtypes = [vp, vp, vp, vp]
    L.ma_read_window_row.argtypes = [vp, C.c_int64, vp, vp]
    L.ma_read_error_buffer_blocks.argtypes = [vp, C.c_int64, C.c_int64, vp, vp, vp]
    L.ma_read_window_blocks.argtypes = [vp, C.c_int64, C.c_int64, C.c_int64, vp, vp]
    L.ma_read_error_vector.argtypes = [vp, vp]
    L.ma_write_state.argtypes = [vp, vp, vp, vp, C.c_int64, C.c_int64, vp, vp, vp]
    L.ma_set_params.argtypes = [vp, vp]
    L.ma_save_checkpoint.argtypes = [vp, vp, C.c_int32, C.c_char_p]
    L.ma_step_front.argtypes = [vp, vp, C.c_int64, C.c_int64, vp, vp, vp]
    L.ma_scatter_rows.argtypes = [vp, vp, vp, C.c_int64, C.c_int64, vp]
    L.ma_step_stats.argtypes = [vp, vp, C.c_double, vp]
    L.ma_load_checkpoint.argtypes = [vp, vp, C.c_int32, C.c_char_p]
    L.ma_get_layout.argtypes = [vp, P(Layout)]
    L.ma_kernel_launches.argtypes = [vp]
    L.ma_kernel_launches.restype = C.c_int64
    L.ma_debug_counters.argtypes = [vp, P(C.c_int64), C.c_int]
    L.ma_last_error.restype = C.c_char_p
    L.ma_last_error.argtypes = []
    L.ma_version.restype = C.c_char_p
    L.ma_version.argtypes = []
    L.ma_fill_synthetic.argtypes = [vp, C.c_int32, C.c_int64, C.c_uint64, C.c_uint64, C.c_int64,
                                    C.c_int32, vp]
    for name in EXPORTED:
        fn = getattr(L, name)
        if fn.restype is C.c_int:  # default restype -> ma_status
            fn.restype = C.c_int
    _lib = L
    return L


def check(status: int) -> None:
    if status != MA_OK:
        raise MicroAdamError(status, lib().ma_last_error().decode())


def default_config() -> Config:
    cfg = Config()
    lib().ma_config_default(C.byref(cfg))
    return cfg
