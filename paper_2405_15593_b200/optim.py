"""Host-side mirror of the reference optimizer interface over the C ABI.

Reference (paths under /root/reference/proj)      -> here
  microadam::HyperParams        optim.hpp:15-30      HyperParams
  microadam::StepReport         optim.hpp:32-38      StepReport
  microadam::MicroAdamOptimizer optim.hpp:98-128     MicroAdamOptimizer (host vectors, fp64,
                                                     bit-identical to the reference step)
  microadam::GradientWindow     window.hpp:10-33     GradientWindow (read back from device)
  microadam::QuantizedErrorBuffer quantize.hpp:54-70 QuantizedErrorBuffer (read back)
  the north-star device engine                      MicroAdam: construct from parameter count +
                                                     block/density/window/quant settings, then
                                                     step(params, grads, lr) on device tensors

Errors mirror the reference's throw sites: invalid configs, dimension
mismatch and non-finite gradients raise ValueError (std::invalid_argument);
error_buffer() on a lossless engine raises RuntimeError (std::logic_error).
torch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _capi
from ._capi import check, lib

_NP_DTYPE = {"f64": np.float64, "f32": np.float32}


class InvalidArgument(ValueError):
    pass


def _raise(status: int) -> None:
    msg = lib().ma_last_error().decode()
    if status in (_capi.MA_ERR_INVALID_ARG, _capi.MA_ERR_DIM, _capi.MA_ERR_NONFINITE):
        raise InvalidArgument(msg)
    if status == _capi.MA_ERR_STATE:
        raise RuntimeError(msg)
    raise _capi.MicroAdamError(status, msg)


def _ok(status: int) -> None:
    if status != _capi.MA_OK:
        _raise(status)


@dataclass
class HyperParams:
    """optim.hpp:15-30 (same defaults)."""
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    lr: float = 1e-3
    weight_decay: float = 0.0
    window: int = 10
    density: float = 0.01
    k: Optional[int] = None
    bits: int = 4
    block: int = 4096
    bucket: int = 64

    def to_c(self) -> _capi.Hyper:
        h = _capi.Hyper()
        h.beta1, h.beta2, h.eps, h.lr = self.beta1, self.beta2, self.eps, self.lr
        h.weight_decay, h.window, h.density = self.weight_decay, self.window, self.density
        h.k = self.k if self.k is not None else 0
        h.bits, h.block, h.bucket = self.bits, self.block, self.bucket
        return h

    def validate(self) -> None:
        """optim.cpp:7-21."""
        cfg = _capi.default_config()
        cfg.hp = self.to_c()
        st = lib().ma_validate(C.byref(cfg), self.k if self.k else 1)
        if st == _capi.MA_ERR_INVALID_ARG:
            _raise(st)

    def resolve_k(self, dim: int) -> int:
        """optim.cpp:23-30."""
        if self.k is not None:
            if self.k > dim:
                raise InvalidArgument("HyperParams: k exceeds dimension")
            return self.k
        return max(1, min(dim, math.ceil(self.density * float(dim))))

    @staticmethod
    def from_any(hp) -> "HyperParams":
        if hp is None:
            return HyperParams()
        if isinstance(hp, HyperParams):
            return hp
        return HyperParams(**hp)


@dataclass
class StepReport:
    """optim.hpp:32-38."""
    grad_norm: float = 0.0
    error_norm: float = 0.0
    empirical_q: float = 0.0
    update_nnz: int = 0
    loss: float = 0.0

    @staticmethod
    def from_c(r: _capi.Report) -> "StepReport":
        return StepReport(r.grad_norm, r.error_norm, r.empirical_q, int(r.update_nnz), r.loss)


@dataclass
class SparseSelection:
    """compress.hpp:9-17."""
    dim: int = 0
    indices: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def size(self) -> int:
        return int(self.indices.size)


@dataclass
class GradientWindow:
    """window.hpp:10-33, rows in the reference's slot-major global-index layout."""
    dim: int
    capacity: int
    row_width: int
    head: int
    filled: int
    step: int
    stamps: np.ndarray
    indices: np.ndarray  # [capacity, row_width] int64 (zeros for unwritten rows)
    values: np.ndarray   # [capacity, row_width] float64


@dataclass
class QuantizedErrorBuffer:
    """quantize.hpp:54-70: packed codes (low nibble first) + per-bucket (lo, hi)."""
    dim: int
    bits: int
    bucket: int
    codes: np.ndarray
    lo: np.ndarray
    hi: np.ndarray

    def num_buckets(self) -> int:
        return (self.dim + self.bucket - 1) // self.bucket

    def decode(self) -> np.ndarray:
        """quantize.cpp:164-178 (separate multiply and add, fp64)."""
        # LSB-first bit stream of `bits`-wide codes (quantize.cpp:102-128)
        bitstream = np.unpackbits(self.codes, bitorder="little")
        pos = np.arange(self.dim, dtype=np.int64)[:, None] * self.bits + np.arange(self.bits)[None, :]
        weights = (1 << np.arange(self.bits, dtype=np.int64))[None, :]
        codes = (bitstream[pos].astype(np.int64) * weights).sum(axis=1).astype(np.float64)
        b = np.arange(self.dim) // self.bucket
        lvl = np.where(self.lo == self.hi, 0.0, (self.hi - self.lo) / float((1 << self.bits) - 1))
        return codes * lvl[b] + self.lo[b]


def _make_config(hp: HyperParams, blockwise: bool, lossless: bool, param_dtype: str,
                 grad_dtype: str, value_dtype: str, finite_mode: str) -> _capi.Config:
    cfg = _capi.default_config()
    cfg.hp = hp.to_c()
    cfg.blockwise = int(blockwise)
    cfg.lossless_error = int(lossless)
    cfg.param_dtype = _capi.DTYPE_CODES[param_dtype]
    cfg.grad_dtype = _capi.DTYPE_CODES[grad_dtype]
    cfg.value_dtype = _capi.DTYPE_CODES[value_dtype]
    cfg.finite_mode = {"flag": _capi.MA_FINITE_FLAG, "strict": _capi.MA_FINITE_STRICT,
                       "off": _capi.MA_FINITE_OFF}[finite_mode]
    return cfg


def layout(dim: int, hp=None, *, blockwise: bool = True, block_range=(0, -1),
           value_dtype: str = "bf16") -> _capi.Layout:
    """Derived layout without touching a device (optim.cpp:137-144)."""
    hp = HyperParams.from_any(hp)
    cfg = _make_config(hp, blockwise, False, "f32", "f32", value_dtype, "flag")
    out = _capi.Layout()
    _ok(lib().ma_layout(C.byref(cfg), dim, block_range[0], block_range[1], C.byref(out)))
    return out


class _Handle:
    """Owns one ma_handle and its state readers."""

    def __init__(self, cfg: _capi.Config, dim: int, device: int, block_range=(0, -1)):
        self._h = C.c_void_p()
        _ok(lib().ma_create_shard(C.byref(cfg), dim, block_range[0], block_range[1], device,
                                  C.byref(self._h)))
        self.cfg = cfg
        self.global_dim = dim
        lay = _capi.Layout()
        _ok(lib().ma_get_layout(self._h, C.byref(lay)))
        self.layout = lay
        self.m = cfg.hp.window

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            lib().ma_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def counters(self):
        s, hd, f = C.c_int64(), C.c_int64(), C.c_int64()
        stamps = (C.c_int64 * self.m)()
        _ok(lib().ma_get_counters(self._h, C.byref(s), C.byref(hd), C.byref(f), stamps))
        return s.value, hd.value, f.value, np.array(stamps[:], np.int64)

    def window(self) -> GradientWindow:
        step, head, filled, stamps = self.counters()
        rw = self.layout.row_width
        idx = np.zeros((self.m, rw), np.int64)
        val = np.zeros((self.m, rw), np.float64)
        for r in range(self.m):
            if stamps[r] == 0:
                continue
            _ok(lib().ma_read_window_row(self._h, r, idx[r].ctypes.data, val[r].ctypes.data))
        return GradientWindow(self.layout.dim, self.m, rw, head, filled, step, stamps, idx, val)

    def error_buffer(self) -> QuantizedErrorBuffer:
        lay = self.layout
        codes = np.zeros(lay.code_bytes, np.uint8)
        lo = np.zeros(lay.num_buckets)
        hi = np.zeros(lay.num_buckets)
        _ok(lib().ma_read_error_buffer(self._h, codes.ctypes.data, lo.ctypes.data, hi.ctypes.data))
        return QuantizedErrorBuffer(lay.dim, self.cfg.hp.bits, self.cfg.hp.bucket, codes, lo, hi)

    def error_buffer_blocks(self, block_begin: int, block_end: int):
        """error_buffer() of blocks [block_begin, block_end): (codes, lo, hi)."""
        lay = self.layout
        e0 = block_begin * lay.block
        e1 = min(lay.dim, block_end * lay.block)
        bits, bucket = self.cfg.hp.bits, self.cfg.hp.bucket
        codes = np.zeros((e1 * bits + 7) // 8 - (e0 * bits) // 8, np.uint8)
        nq = (e1 + bucket - 1) // bucket - e0 // bucket
        lo = np.zeros(nq)
        hi = np.zeros(nq)
        _ok(lib().ma_read_error_buffer_blocks(self._h, block_begin, block_end, codes.ctypes.data,
                                              lo.ctypes.data, hi.ctypes.data))
        return codes, lo, hi

    def window_blocks(self, slot: int, block_begin: int, block_end: int):
        """window().rows[slot] restricted to blocks [block_begin, block_end): (indices, values)."""
        lay = self.layout
        n = 0
        for b in range(block_begin, block_end):
            n += min(lay.per_block_k, min(lay.block, lay.dim - b * lay.block))
        idx = np.zeros(n, np.int64)
        val = np.zeros(n, np.float64)
        _ok(lib().ma_read_window_blocks(self._h, slot, block_begin, block_end, idx.ctypes.data,
                                        val.ctypes.data))
        return idx, val

    def write_state(self, codes, lo, hi, step, head, stamps, win_idx, win_val) -> None:
        a = [np.ascontiguousarray(codes, np.uint8), np.ascontiguousarray(lo, np.float64),
             np.ascontiguousarray(hi, np.float64), np.ascontiguousarray(stamps, np.int64),
             np.ascontiguousarray(win_idx, np.int64), np.ascontiguousarray(win_val, np.float64)]
        _ok(lib().ma_write_state(self._h, a[0].ctypes.data, a[1].ctypes.data, a[2].ctypes.data,
                                 int(step), int(head), a[3].ctypes.data, a[4].ctypes.data,
                                 a[5].ctypes.data))

    def kernel_launches(self) -> int:
        return int(lib().ma_kernel_launches(self._h))

    def debug_counters(self) -> dict:
        """Fast-kernel diagnostics (needs MA_DEBUG_COUNTERS=1 at creation)."""
        out = (C.c_int64 * 20)()
        _ok(lib().ma_debug_counters(self._h, out, 20))
        return {"select_fallback_blocks": out[0], "exact_quotient_elems": out[1],
                "threshold_misses": out[2], "threshold_too_low": out[3],
                "dup_list_overflow_blocks": out[4], "dup_entries": out[5],
                "threshold_refinements": out[6], "tie_ranks": out[7],
                "phase_cycles": list(out[8:20])}


_TORCH_DTYPE_NAMES = {"torch.float64": "f64", "torch.float32": "f32", "torch.bfloat16": "bf16"}


class MicroAdam(_Handle):
    """Device engine: MicroAdam(dim, hp, ...) then step(params, grads, lr).

    ``params`` / ``grads`` are CUDA tensors (or raw device pointers) covering the
    engine's block range; θ is updated in place on ``stream`` (default: torch's
    current stream), asynchronously unless ``report=True``.
    """

    def __init__(self, dim: int, hp=None, *, param_dtype: str = "f32", grad_dtype: str = "f32",
                 value_dtype: str = "bf16", finite_mode: str = "flag", device: int = 0,
                 blockwise: bool = True, block_range=(0, -1)):
        self.hp = HyperParams.from_any(hp)
        self.param_dtype, self.grad_dtype, self.value_dtype = param_dtype, grad_dtype, value_dtype
        cfg = _make_config(self.hp, blockwise, False, param_dtype, grad_dtype, value_dtype,
                           finite_mode)
        super().__init__(cfg, dim, device, block_range)
        self.device = device

    def _ptr(self, t, want: str, what: str) -> int:
        if isinstance(t, int):
            return t
        name = _TORCH_DTYPE_NAMES.get(str(t.dtype))
        if name != want:
            raise InvalidArgument(f"{what}: dtype {t.dtype} does not match configured {want}")
        if t.numel() != self.layout.dim:
            raise InvalidArgument("step: gradient dim mismatch" if what == "grads"
                                  else "step: parameter dim mismatch")
        if not t.is_cuda or not t.is_contiguous():
            raise InvalidArgument(f"{what}: expected a contiguous CUDA tensor")
        return t.data_ptr()

    def step(self, params, grads, lr: Optional[float] = None, stream=None,
             report: bool = False) -> Optional[StepReport]:
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(self.device).cuda_stream
        elif hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        rep = _capi.Report()
        _ok(lib().ma_step(self._h, self._ptr(params, self.param_dtype, "params"),
                          self._ptr(grads, self.grad_dtype, "grads"),
                          self.hp.lr if lr is None else lr, C.c_void_p(stream),
                          C.byref(rep) if report else None))
        return StepReport.from_c(rep) if report else None

    def step_reduce(self, params, grads, sources, scale: float = 1.0, lr: Optional[float] = None,
                    stream=None, report: bool = False) -> Optional[StepReport]:
        """Step with the gradient reduce-scatter fused in (ma_step_reduce).

        `sources` are the ranks' gradients for this engine's element range:
        device tensors of the gradient dtype or raw device pointers (peer
        pointers from symmetric memory / CUDA IPC). The step uses
        g = rn(((s_0 + s_1) + ...) * scale) (fp32 sums for bf16/f32), written
        into `grads` (which may be one of the sources)."""
        if not 1 <= len(sources) <= 8:
            raise ValueError("step_reduce: 1 to 8 gradient sources")
        ptrs = (C.c_void_p * len(sources))(*[
            s if isinstance(s, int) else self._ptr(s, self.grad_dtype, "grads") for s in sources])
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(self.device).cuda_stream
        elif hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        rep = _capi.Report()
        _ok(lib().ma_step_reduce(self._h, self._ptr(params, self.param_dtype, "params"),
                                 self._ptr(grads, self.grad_dtype, "grads"), ptrs, len(sources),
                                 float(scale), self.hp.lr if lr is None else lr, C.c_void_p(stream),
                                 C.byref(rep) if report else None))
        return StepReport.from_c(rep) if report else None

    def step_allgather(self, params_full, grads, comm: "Comm", lr: Optional[float] = None, stream=None,
                       report: bool = False) -> Optional[StepReport]:
        """ZeRO-1 data-parallel step (ma_step_allgather): this shard engine steps
        its slice of the full θ replica `params_full`, then NCCL all-gathers the
        updated shards into every rank's replica. `params_full` holds dim
        elements (grouped broadcasts) or nranks * shard stride (one all-gather);
        `grads` covers this engine's blocks only."""
        rep = _capi.Report()
        n = params_full.numel() if hasattr(params_full, "numel") else int(params_full[1])
        ptr = params_full.data_ptr() if hasattr(params_full, "data_ptr") else int(params_full[0])
        _ok(lib().ma_step_allgather(self._h, ptr, n, self._ptr(grads, self.grad_dtype, "grads"),
                                    self.hp.lr if lr is None else lr, comm.handle,
                                    C.c_void_p(self._stream(stream)), C.byref(rep) if report else None))
        return StepReport.from_c(rep) if report else None

    def allgather_params(self, params_full, comm: "Comm", stream=None) -> None:
        """The all-gather half of step_allgather (ma_allgather_params)."""
        _ok(lib().ma_allgather_params(self._h, params_full.data_ptr(), params_full.numel(), comm.handle,
                                      C.c_void_p(self._stream(stream))))

    def exchange_rows(self, stage, rows, comm: "Comm", stream=None) -> None:
        """Sparse propagation's exchange (ma_exchange_rows): NCCL all-gather of every
        rank's stage rows into `rows`, then scatter them into this step's window slot."""
        kbs = self.layout.kb_stride
        _ok(lib().ma_exchange_rows(self._h, stage[0].data_ptr(), stage[1].data_ptr(), stage[0].numel() // kbs,
                                   rows[0].data_ptr(), rows[1].data_ptr(), comm.handle,
                                   C.c_void_p(self._stream(stream))))

    def step_host(self, h_params, h_grads, lr: Optional[float] = None,
                  report: bool = False) -> Optional[StepReport]:
        """Reference-facing host path (ma_step_host): host θ in/out, host g in.

        Buffers are CPU tensors (pinned for full overlap), numpy arrays or raw
        host pointers of the configured dtypes. Returns once h_params holds
        the updated θ."""
        def hptr(x):
            if isinstance(x, int):
                return x
            if isinstance(x, np.ndarray):
                return x.ctypes.data
            return x.data_ptr()
        rep = _capi.Report()
        _ok(lib().ma_step_host(self._h, hptr(h_params), hptr(h_grads),
                               self.hp.lr if lr is None else lr,
                               C.byref(rep) if report else None))
        return StepReport.from_c(rep) if report else None

    def set_params(self, h_params) -> None:
        ptr = h_params if isinstance(h_params, int) else (
            h_params.ctypes.data if isinstance(h_params, np.ndarray) else h_params.data_ptr())
        _ok(lib().ma_set_params(self._h, ptr))

    def synchronize(self) -> None:
        _ok(lib().ma_sync(self._h))

    def step_count(self) -> int:
        return self.counters()[0]

    # -- sparse parameter propagation (ma_step_front / ma_scatter_rows / ma_step_stats) --
    def stage_buffers(self, nblocks: int):
        """Device (idx, values) stage buffers for `nblocks` blocks' window rows."""
        import torch
        kbs = self.layout.kb_stride
        vt = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[self.value_dtype]
        return (torch.empty(nblocks * kbs, dtype=torch.int16, device=f"cuda:{self.device}"),
                torch.empty(nblocks * kbs, dtype=vt, device=f"cuda:{self.device}"))

    def _stream(self, stream):
        if stream is None:
            import torch
            return torch.cuda.current_stream(self.device).cuda_stream
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else stream

    def step_front(self, grads, block_begin: int, block_end: int, stage, stream=None) -> None:
        """EF decode, Top-K, window row (also into `stage`) and EF re-quantization
        for blocks [block_begin, block_end); `grads` covers exactly that range."""
        _ok(lib().ma_step_front(self._h, grads.data_ptr(), block_begin, block_end, stage[0].data_ptr(),
                                stage[1].data_ptr(), C.c_void_p(self._stream(stream))))

    def scatter_rows(self, rows, block_begin: int, block_end: int, stream=None) -> None:
        """Put the (gathered) rows of blocks [block_begin, block_end) into this step's window slot."""
        _ok(lib().ma_scatter_rows(self._h, rows[0].data_ptr(), rows[1].data_ptr(), block_begin, block_end,
                                  C.c_void_p(self._stream(stream))))

    def step_stats(self, params, lr: Optional[float] = None, stream=None) -> None:
        """ADAM_STATS + θ update over all blocks into `params` (this rank's replica)."""
        _ok(lib().ma_step_stats(self._h, self._ptr(params, self.param_dtype, "params"),
                                self.hp.lr if lr is None else lr, C.c_void_p(self._stream(stream))))

    def save_checkpoint(self, path: str, params) -> None:
        """save_checkpoint (checkpoint.cpp:50-86): the reference's MADM v1 file
        from this engine's state and θ (a CUDA tensor of the param dtype, or a
        host numpy array / CPU tensor)."""
        on_dev, ptr = _buffer(params)
        _ok(lib().ma_save_checkpoint(self._h, ptr, on_dev, os.fsencode(path)))

    def load_checkpoint(self, path: str, params=None) -> None:
        """Restore state (and θ into `params` when given) from a MADM v1 file
        (checkpoint.cpp:88-140 format), e.g. one written by the reference."""
        on_dev, ptr = _buffer(params) if params is not None else (0, None)
        _ok(lib().ma_load_checkpoint(self._h, ptr, on_dev, os.fsencode(path)))


class Comm:
    """An NCCL communicator owned through the C ABI (ma_comm_*): rank 0 calls
    unique_id(), every rank receives those 128 bytes (any channel, e.g.
    torch.distributed.broadcast_object_list) and builds Comm(id, nranks, rank, device)."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int = 0):
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _ok(lib().ma_comm_init(buf, nranks, rank, device, C.byref(h)))
        self.handle = h
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _ok(lib().ma_comm_unique_id(buf))
        return bytes(buf)

    def close(self) -> None:
        if getattr(self, "handle", None):
            _ok(lib().ma_comm_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _buffer(x):
    """(on_device, pointer) of a CUDA tensor, CPU tensor or numpy array."""
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise InvalidArgument("checkpoint: expected a contiguous array")
        return 0, x.ctypes.data
    if not x.is_contiguous():
        raise InvalidArgument("checkpoint: expected a contiguous tensor")
    return (1 if x.is_cuda else 0), x.data_ptr()


class MicroAdamOptimizer(_Handle):
    """Drop-in for microadam::MicroAdamOptimizer(theta0, hp, blockwise=false,
    lossless_error=false) (optim.hpp:98-128, same defaults as optim.hpp:103-104): host fp64 vectors in and out, fp64 on the device,
    reject-before-mutate finiteness — bit-identical to the reference step."""

    def __init__(self, theta0, hp=None, blockwise: bool = False, lossless_error: bool = False,
                 device: int = 0):
        self.hp = HyperParams.from_any(hp)
        self._theta = np.array(theta0, dtype=np.float64, copy=True)
        cfg = _make_config(self.hp, blockwise, lossless_error, "f64", "f64", "f64", "strict")
        super().__init__(cfg, self._theta.size, device)
        _ok(lib().ma_set_params(self._h, self._theta.ctypes.data))
        self._last = SparseSelection(self._theta.size)

    def step(self, grad) -> StepReport:
        g = np.ascontiguousarray(grad, dtype=np.float64)
        if g.size != self._theta.size:
            raise InvalidArgument("step: gradient dim mismatch")
        rep = _capi.Report()
        _ok(lib().ma_step_host(self._h, self._theta.ctypes.data, g.ctypes.data, self.hp.lr,
                               C.byref(rep)))
        _, head, _, _ = self.counters()
        slot = (head + self.m - 1) % self.m
        rw = self.layout.row_width
        idx = np.zeros(rw, np.int64)
        val = np.zeros(rw)
        _ok(lib().ma_read_window_row(self._h, slot, idx.ctypes.data, val.ctypes.data))
        self._last = SparseSelection(self._theta.size, idx, val)
        return StepReport.from_c(rep)

    def params(self) -> np.ndarray:
        return self._theta

    def name(self) -> str:
        return "microadam"

    def lossless(self) -> bool:
        return bool(self.cfg.lossless_error)

    def error_vector(self) -> np.ndarray:
        """error_vector() (optim.cpp:160-162): decoded EF, or the dense residual."""
        out = np.zeros(self.layout.dim)
        _ok(lib().ma_read_error_vector(self._h, out.ctypes.data))
        return out

    def last_selection(self) -> SparseSelection:
        return self._last

    def save_checkpoint(self, path: str) -> None:
        """save_checkpoint(path, opt) (checkpoint.hpp:28-33): the MADM v1 file."""
        _ok(lib().ma_save_checkpoint(self._h, self._theta.ctypes.data, 0, os.fsencode(path)))

    def load_checkpoint(self, path: str) -> None:
        """Resume from a MADM v1 file (θ into params(), state into the device)."""
        _ok(lib().ma_load_checkpoint(self._h, self._theta.ctypes.data, 0, os.fsencode(path)))

    def step_count(self) -> int:
        return self.counters()[0]

    def hyper(self) -> HyperParams:
        return self.hp
