"""Tiny tile-kernel run for compute-sanitizer (racecheck / synccheck / memcheck)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.tile_check import run  # noqa: E402
import oracle  # noqa: E402

oracle.build()
run(12, 0, dict(lr=1e-3, window=4), "bf16", 6, 2)
run(6, 0, dict(lr=1e-3, density=0.05, window=6), "bf16", 8, 2)
