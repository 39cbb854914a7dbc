#!/usr/bin/env python
"""Time the fused step at several vector sizes (diagnostic, not a bench line)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_15593_b200 as ma  # noqa: E402

sizes = [int(float(x)) for x in (sys.argv[1:] or ["1.1e8", "4.4e8", "1.3e9", "3e9", "6.738415616e9"])]
L = ma.lib()
s = torch.cuda.current_stream().cuda_stream
for d in sizes:
    eng = ma.MicroAdam(d, dict(), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
    p = torch.empty(d, dtype=torch.bfloat16, device="cuda")
    g = torch.empty(d, dtype=torch.bfloat16, device="cuda")
    ma._capi.check(L.ma_fill_synthetic(p.data_ptr(), 2, d, 1, 0, 0, 0, s))
    times = []
    dbgon = os.environ.get("MA_DEBUG_COUNTERS") == "1"
    prev = None
    per = []
    for i in range(int(os.environ.get("SCAN_STEPS", "12"))):
        cyc = int(os.environ.get("SCAN_CYCLE", "0"))  # >0: gradients repeat with this period (bench.py)
        ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), 2, d, 42, (i % cyc if cyc else i) + 1, 0, 0, s))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.step(p, g, 1e-3)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        if dbgon:
            cur = eng.debug_counters()
            if prev is not None:
                per.append({k: cur[k] - prev[k] for k in cur if k != "phase_cycles"})
            prev = cur
    t = sorted(times[6:])[len(times[6:]) // 2]
    dbg = eng.debug_counters() if os.environ.get("MA_DEBUG_COUNTERS") == "1" else {}
    print(f"d={d:>12,}  step {t:9.3f} ms  {d / t / 1e6:8.3f} Gparam/s  {7.9 * d / t / 1e6:8.1f} GB/s  "
          f"steps: {' '.join(f'{x:.2f}' for x in times)} {dbg}", flush=True)
    nb = d // 4096
    for i, c in enumerate(per):
        print(f"   step {i + 2:3d}: misses {c['threshold_misses'] / nb:6.3f}  too_low {c['threshold_too_low'] / nb:6.3f}"
              f"  exactq/blk {c['exact_quotient_elems'] / nb:6.2f}  fallback {c['select_fallback_blocks']}"
              f"  flagged/blk {c['select_fallback_blocks'] / nb:7.2f}  refine {c['threshold_refinements'] / nb:6.3f}  dup/blk {c['dup_entries'] / nb:6.1f}  dup-overflow {c['dup_list_overflow_blocks'] / nb:6.3f}")
    del eng, p, g
    torch.cuda.empty_cache()
