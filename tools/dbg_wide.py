import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2405_15593_b200 as ma
d = 4096 * 60000
L = ma.lib(); s = torch.cuda.current_stream().cuda_stream
for dens in (0.02, 0.05):
    eng = ma.MicroAdam(d, dict(density=dens, window=10), param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16")
    p = torch.empty(d, dtype=torch.bfloat16, device="cuda"); g = torch.empty(d, dtype=torch.bfloat16, device="cuda")
    ma._capi.check(L.ma_fill_synthetic(p.data_ptr(), 2, d, 1, 0, 0, 0, s))
    prev = None
    for i in range(14):
        ma._capi.check(L.ma_fill_synthetic(g.data_ptr(), 2, d, 42, i + 1, 0, 0, s))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); eng.step(p, g, 1e-3); e1.record(); torch.cuda.synchronize()
        c = eng.debug_counters()
        if prev:
            dd = {k: c[k] - prev[k] for k in c if k != "phase_cycles"}
            nb = d // 4096
            print(f"dens {dens} step {i+1}: {e0.elapsed_time(e1):7.2f} ms  slow {dd['threshold_misses']/nb:.3f} overfull {dd['threshold_too_low']/nb:.3f} refine {dd['threshold_refinements']/nb:.3f} dup/blk {dd['dup_entries']/nb:.1f} dupovf {dd['dup_list_overflow_blocks']/nb:.3f} ties {dd['tie_ranks']/nb:.3f} exactq {dd['exact_quotient_elems']/nb:.2f}")
        prev = c
    del eng, p, g; torch.cuda.empty_cache()
