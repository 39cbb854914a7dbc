"""paper_2405_15593_b200 — B200-native (sm_100a) MicroAdam optimizer step.

The per-step hot path (EF decode + accumulate, block Top-K, 4-bit EF
re-quantization, window-ring write, ADAM_STATS + update) runs in one fused
CUDA kernel in libmicroadam_cuda.so, behind the C ABI of
include/microadam_cuda.h. This package is the host-side mirror of the
reference optimizer interface (see optim.py) on that ABI; there is no CPU
fallback.
"""
from ._capi import LIB_PATH, MicroAdamError, lib
from .optim import (Comm, GradientWindow, HyperParams, InvalidArgument, MicroAdam, MicroAdamOptimizer,
                    QuantizedErrorBuffer, SparseSelection, StepReport, layout)

__all__ = [
    "LIB_PATH", "MicroAdamError", "lib", "Comm", "GradientWindow", "HyperParams", "InvalidArgument",
    "MicroAdam", "MicroAdamOptimizer", "QuantizedErrorBuffer", "SparseSelection", "StepReport",
    "layout",
]
