"""CPU checkers for the MicroAdam step — TEST INFRASTRUCTURE ONLY.

Two checkers, both loaded through ctypes:

* ``Oracle``     — oracle/microadam_oracle.c, the C restatement of the reference
                   blockwise step (each function cites the reference file:line).
* ``Reference``  — oracle/_ref/libmicroadam_ref.so, the UNMODIFIED reference
                   sources (/root/reference/proj/src) compiled by oracle/Makefile
                   plus the extern "C" shim oracle/ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline. The product package (paper_2405_15593_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmicroadam_ref.so")

F64, F32, BF16 = 0, 1, 2
DTYPES = {"f64": F64, "f32": F32, "bf16": BF16}

_p = np.ctypeslib.ndpointer
_f64 = _p(dtype=np.float64, flags="C_CONTIGUOUS")
_i64 = _p(dtype=np.int64, flags="C_CONTIGUOUS")
_u8 = _p(dtype=np.uint8, flags="C_CONTIGUOUS")
_u32 = _p(dtype=np.uint32, flags="C_CONTIGUOUS")


def build(force: bool = False) -> None:
    """Build the checkers (the reference leg only where /root/reference exists)."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    if force or not os.path.exists(ORACLE_SO) or (
        "ref" in targets and not os.path.exists(REF_SO)
    ):
        subprocess.check_call(["make", "-s", "-C", HERE] + targets)


class _Report(C.Structure):
    _fields_ = [
        ("grad_norm", C.c_double),
        ("error_norm", C.c_double),
        ("empirical_q", C.c_double),
        ("update_nnz", C.c_int64),
        ("loss", C.c_double),
    ]


_olib = None
_rlib = None


def oracle_lib():
    global _olib
    if _olib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.mo_create.restype = C.c_void_p
        L.mo_create.argtypes = [C.c_int64, _f64, C.c_double, C.c_double, C.c_double, C.c_double,
                                C.c_int64, C.c_double, C.c_int64, C.c_int, C.c_int64, C.c_int64,
                                C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.mo_destroy.argtypes = [C.c_void_p]
        L.mo_step.restype = C.c_int
        L.mo_step.argtypes = [C.c_void_p, _f64, C.c_double, C.POINTER(_Report)]
        for name in ("mo_dim", "mo_row_width", "mo_per_block_k_of", "mo_block_of", "mo_num_buckets"):
            getattr(L, name).restype = C.c_int64
            getattr(L, name).argtypes = [C.c_void_p]
        for name, ty in (("mo_params", C.c_double), ("mo_codes", C.c_uint8), ("mo_lo", C.c_double),
                         ("mo_hi", C.c_double), ("mo_last_idx", C.c_int64), ("mo_last_val", C.c_double),
                         ("mo_stamps", C.c_int64), ("mo_win_idx", C.c_int64), ("mo_win_val", C.c_double)):
            getattr(L, name).restype = C.POINTER(ty)
            getattr(L, name).argtypes = [C.c_void_p]
        L.mo_counters.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int64)]
        L.mo_bf16_round.restype = C.c_double
        L.mo_bf16_round.argtypes = [C.c_double]
        L.mo_round.restype = C.c_double
        L.mo_round.argtypes = [C.c_double, C.c_int]
        L.mo_per_block_k.restype = C.c_int64
        L.mo_per_block_k.argtypes = [C.c_int64, C.c_double]
        L.mo_topk_blockwise.restype = C.c_int64
        L.mo_topk_blockwise.argtypes = [_f64, C.c_int64, C.c_int64, C.c_int64, _i64, _f64]
        L.mo_topk_global.restype = C.c_int64
        L.mo_topk_global.argtypes = [_f64, C.c_int64, C.c_int64, _i64, _f64]
        L.mo_level.restype = C.c_double
        L.mo_level.argtypes = [C.c_double, C.c_double, C.c_int]
        L.mo_quant_params.argtypes = [_f64, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.mo_quantize_nearest.restype = C.c_uint32
        L.mo_quantize_nearest.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int]
        L.mo_pack.argtypes = [_u32, C.c_int64, C.c_int, _u8]
        L.mo_unpack.argtypes = [_u8, C.c_int64, C.c_int, _u32]
        L.mo_encode.argtypes = [_f64, C.c_int64, C.c_int, C.c_int64, _u8, _f64, _f64]
        L.mo_decode.argtypes = [_u8, _f64, _f64, C.c_int64, C.c_int, C.c_int64, _f64]
        L.mo_adam_stats.argtypes = [_i64, _f64, _i64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                    C.c_int64, C.c_double, C.c_int, _f64]
        L.mo_synth_fill.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int, C.c_int, _f64]
        _olib = L
    return _olib


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _rlib
    if _rlib is None:
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise RuntimeError("oracle/_ref/libmicroadam_ref.so not built (needs /root/reference)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_create.restype = C.c_void_p
        L.ref_create.argtypes = [C.c_int64, _f64, C.c_double, C.c_double, C.c_double, C.c_double,
                                 C.c_int64, C.c_double, C.c_int64, C.c_int, C.c_int64, C.c_int64,
                                 C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.ref_destroy.argtypes = [C.c_void_p]
        L.ref_step.restype = C.c_int
        L.ref_step.argtypes = [C.c_void_p, _f64, C.c_int64, _f64]
        L.ref_dim.restype = C.c_int64
        L.ref_dim.argtypes = [C.c_void_p]
        L.ref_params.argtypes = [C.c_void_p, _f64]
        L.ref_row_width.restype = C.c_int64
        L.ref_row_width.argtypes = [C.c_void_p]
        L.ref_counters.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int64), _i64]
        L.ref_window_row.restype = C.c_int64
        L.ref_window_row.argtypes = [C.c_void_p, C.c_int64, _i64, _f64]
        L.ref_last_selection.restype = C.c_int64
        L.ref_last_selection.argtypes = [C.c_void_p, _i64, _f64]
        L.ref_num_buckets.restype = C.c_int64
        L.ref_num_buckets.argtypes = [C.c_void_p]
        L.ref_error_buffer.restype = C.c_int
        L.ref_error_buffer.argtypes = [C.c_void_p, _u8, _f64, _f64]
        L.ref_error_vector.argtypes = [C.c_void_p, _f64]
        L.ref_topk_blockwise.restype = C.c_int64
        L.ref_topk_blockwise.argtypes = [_f64, C.c_int64, C.c_int64, C.c_int64, _i64, _f64]
        L.ref_topk_global.restype = C.c_int64
        L.ref_topk_global.argtypes = [_f64, C.c_int64, C.c_int64, _i64, _f64]
        L.ref_per_block_k.restype = C.c_int64
        L.ref_per_block_k.argtypes = [C.c_int64, C.c_int64, C.c_double]
        L.ref_encode.restype = C.c_int
        L.ref_encode.argtypes = [_f64, C.c_int64, C.c_int, C.c_int64, _u8, _f64, _f64, _f64]
        L.ref_decode.restype = C.c_int
        L.ref_decode.argtypes = [_u8, _f64, _f64, C.c_int64, C.c_int, C.c_int64, _f64]
        L.ref_adam_stats.restype = C.c_int
        L.ref_adam_stats.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, _i64, _f64,
                                     C.c_double, C.c_int, _f64]
        L.ref_save_checkpoint.restype = C.c_int
        L.ref_save_checkpoint.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_load_checkpoint.restype = C.c_int
        L.ref_load_checkpoint.argtypes = [C.c_char_p, _i64, C.c_void_p]
        L.ref_time_shards.restype = C.c_double
        L.ref_time_shards.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int64,
                                      C.c_int64, C.c_double, C.c_int64, _f64]
        _rlib = L
    return _rlib


def ref_load_checkpoint(path: str, dim: int | None = None):
    """The reference's own load_checkpoint (checkpoint.cpp:88-140): raises
    ValueError on what the reference rejects; returns (header dict, θ or None)."""
    L = ref_lib()
    out = np.zeros(6, np.int64)
    theta = np.zeros(dim) if dim else None
    if L.ref_load_checkpoint(os.fsencode(path), out, theta.ctypes.data if theta is not None else None) != 0:
        raise ValueError(L.ref_last_error().decode())
    keys = ("dim", "step", "capacity", "row_width", "head", "filled")
    return dict(zip(keys, (int(x) for x in out))), theta


class State:
    """Snapshot of one optimizer's state in the reference's own layout."""

    def __init__(self, params, codes, lo, hi, step, head, filled, stamps, win_idx, win_val,
                 last_idx, last_val):
        self.params = params
        self.codes = codes
        self.lo = lo
        self.hi = hi
        self.step = step
        self.head = head
        self.filled = filled
        self.stamps = stamps
        self.win_idx = win_idx  # [m, row_width] global int64 (window.hpp:11-15)
        self.win_val = win_val
        self.last_idx = last_idx
        self.last_val = last_val


def _hp_args(hp: dict):
    return (hp.get("beta1", 0.9), hp.get("beta2", 0.999), hp.get("eps", 1e-8), hp.get("lr", 1e-3),
            hp.get("window", 10), hp.get("density", 0.01), hp.get("k", 0) or 0, hp.get("bits", 4),
            hp.get("block", 4096), hp.get("bucket", 64))


class Oracle:
    """C restatement (oracle/microadam_oracle.c) of MicroAdamOptimizer(blockwise=true)."""

    def __init__(self, theta0: np.ndarray, hp: dict | None = None, param_dtype: str = "f64",
                 value_dtype: str = "f64"):
        self.L = oracle_lib()
        hp = dict(hp or {})
        self.hp = hp
        theta0 = np.ascontiguousarray(theta0, dtype=np.float64)
        st = C.c_int(0)
        self.h = self.L.mo_create(theta0.size, theta0, *_hp_args(hp), DTYPES[param_dtype],
                                  DTYPES[value_dtype], C.byref(st))
        if not self.h:
            raise ValueError(f"oracle rejected config (status {st.value})")
        self.dim = theta0.size
        self.m = hp.get("window", 10)
        self.row_width = self.L.mo_row_width(self.h)
        self.per_block_k = self.L.mo_per_block_k_of(self.h)
        self.block = self.L.mo_block_of(self.h)
        self.nbuckets = self.L.mo_num_buckets(self.h)
        self.bits = hp.get("bits", 4)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.mo_destroy(self.h)
            self.h = None

    def step(self, grad: np.ndarray, lr: float | None = None) -> dict:
        grad = np.ascontiguousarray(grad, dtype=np.float64)
        if grad.size != self.dim:
            raise ValueError("step: gradient dim mismatch")
        rep = _Report()
        st = self.L.mo_step(self.h, grad, self.hp.get("lr", 1e-3) if lr is None else lr, C.byref(rep))
        if st != 0:
            raise ValueError(f"step: rejected (status {st})")
        return {"grad_norm": rep.grad_norm, "error_norm": rep.error_norm,
                "empirical_q": rep.empirical_q, "update_nnz": rep.update_nnz}

    def _arr(self, ptr, n, dtype):
        return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)

    def error_vector(self) -> np.ndarray:
        """error_vector() (optim.cpp:160-162)."""
        out = np.zeros(self.dim)
        self.L.ref_error_vector(self.h, out)
        return out

    def save_checkpoint(self, path: str) -> None:
        """The reference's own save_checkpoint (checkpoint.cpp:50-86)."""
        if self.L.ref_save_checkpoint(self.h, os.fsencode(path)) != 0:
            raise ValueError(self.L.ref_last_error().decode())

    def state(self) -> State:
        L, h = self.L, self.h
        s, hd, f = C.c_int64(), C.c_int64(), C.c_int64()
        L.mo_counters(h, C.byref(s), C.byref(hd), C.byref(f))
        nbytes = (self.dim * self.bits + 7) // 8
        rw = self.row_width
        return State(
            self._arr(L.mo_params(h), self.dim, np.float64),
            self._arr(L.mo_codes(h), nbytes, np.uint8),
            self._arr(L.mo_lo(h), self.nbuckets, np.float64),
            self._arr(L.mo_hi(h), self.nbuckets, np.float64),
            s.value, hd.value, f.value,
            self._arr(L.mo_stamps(h), self.m, np.int64),
            self._arr(L.mo_win_idx(h), self.m * rw, np.int64).reshape(self.m, rw),
            self._arr(L.mo_win_val(h), self.m * rw, np.float64).reshape(self.m, rw),
            self._arr(L.mo_last_idx(h), rw, np.int64),
            self._arr(L.mo_last_val(h), rw, np.float64),
        )


class Reference:
    """The unmodified reference MicroAdamOptimizer (optim.hpp:98-128) via ref_shim."""

    def __init__(self, theta0: np.ndarray, hp: dict | None = None, blockwise: bool = True,
                 lossless: bool = False):
        self.L = ref_lib()
        hp = dict(hp or {})
        self.hp = hp
        theta0 = np.ascontiguousarray(theta0, dtype=np.float64)
        st = C.c_int(0)
        self.h = self.L.ref_create(theta0.size, theta0, *_hp_args(hp), int(blockwise), int(lossless),
                                   C.byref(st))
        if not self.h:
            raise ValueError(self.L.ref_last_error().decode())
        self.dim = theta0.size
        self.m = hp.get("window", 10)
        self.bits = hp.get("bits", 4)
        self.row_width = self.L.ref_row_width(self.h)
        self.lossless = lossless

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_destroy(self.h)
            self.h = None

    def step(self, grad: np.ndarray) -> dict:
        grad = np.ascontiguousarray(grad, dtype=np.float64)
        rep = np.zeros(5)
        st = self.L.ref_step(self.h, grad, grad.size, rep)
        if st != 0:
            raise ValueError(self.L.ref_last_error().decode())
        return {"grad_norm": rep[0], "error_norm": rep[1], "empirical_q": rep[2],
                "update_nnz": int(rep[3])}

    def error_vector(self) -> np.ndarray:
        """error_vector() (optim.cpp:160-162)."""
        out = np.zeros(self.dim)
        self.L.ref_error_vector(self.h, out)
        return out

    def save_checkpoint(self, path: str) -> None:
        """The reference's own save_checkpoint (checkpoint.cpp:50-86)."""
        if self.L.ref_save_checkpoint(self.h, os.fsencode(path)) != 0:
            raise ValueError(self.L.ref_last_error().decode())

    def state(self) -> State:
        L, h = self.L, self.h
        s, hd, f = C.c_int64(), C.c_int64(), C.c_int64()
        stamps = np.zeros(self.m, np.int64)
        L.ref_counters(h, C.byref(s), C.byref(hd), C.byref(f), stamps)
        params = np.zeros(self.dim)
        L.ref_params(h, params)
        rw = self.row_width
        win_idx = np.zeros((self.m, rw), np.int64)
        win_val = np.zeros((self.m, rw))
        for r in range(self.m):
            L.ref_window_row(h, r, win_idx[r], win_val[r])
        last_idx = np.zeros(rw, np.int64)
        last_val = np.zeros(rw)
        L.ref_last_selection(h, last_idx, last_val)
        if self.lossless:
            codes = lo = hi = None
        else:
            nb = L.ref_num_buckets(h)
            codes = np.zeros((self.dim * self.bits + 7) // 8, np.uint8)
            lo = np.zeros(nb)
            hi = np.zeros(nb)
            L.ref_error_buffer(h, codes, lo, hi)
        return State(params, codes, lo, hi, s.value, hd.value, f.value, stamps, win_idx, win_val,
                     last_idx, last_val)


def synth(seed: int, step: int, offset: int, n: int, dtype: str = "f64", levels: bool = False,
          heavy: bool = False) -> np.ndarray:
    """The include/ma_synth.h stream, rounded to dtype (float64 array): Gaussian-like,
    16 tie-heavy levels (levels=True) or heavy-tailed per-block-scaled (heavy=True)."""
    out = np.empty(n, np.float64)
    mode = 2 if heavy else (1 if levels else 0)
    oracle_lib().mo_synth_fill(seed, step, offset, n, DTYPES[dtype], mode, out)
    return out


def round_dtype(x: np.ndarray, dtype: str) -> np.ndarray:
    L = oracle_lib()
    return np.array([L.mo_round(float(v), DTYPES[dtype]) for v in np.asarray(x, np.float64).ravel()])
