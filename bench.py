#!/usr/bin/env python
"""Benchmark of the B200 MicroAdam optimizer step (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload llama2-7b|llama2-13b|opt-1.3b|bert-110m|1m]
                    [--density D] [--window M] [--mode shard|allgather|sparse]

A "step" is one MicroAdamOptimizer::step (optim.cpp:164-190) over the whole
workload vector: EF decode + accumulate, block Top-K, 4-bit re-quantization,
window-ring write, ADAM_STATS + update — one fused kernel launch per step.
At N>1 (torchrun, one rank per GPU) the parameter space is block-sharded.
--mode allgather (default, the north star's layout): the 7B vector's blocks
are split over the ranks (paper_2405_15593_b200/sharding.py) and every step
is the rank's shard step followed by the NCCL all-gather of the updated bf16
θ shards into each rank's full replica — ma_step_allgather's two halves
(ma_step + ma_allgather_params) through the C ABI on the library's own NCCL
communicator (strong scaling; step_only and the collective's GB/s are in the
same line). --mode sparse: the EF / Top-K front is sharded, the new window
rows are all-gathered (ma_exchange_rows) and ADAM_STATS + update run on every
rank's replica. --mode shard: rank r steps its own 7B-sized block range of an
N x 7B vector with no collective (weak scaling). Every timed step runs with a
full window: max(W, m) untimed steps come first.

Default workload = BASELINE.json configs[3] (Llama-2-7B-sized vector,
6,738,415,616 params, bf16 θ/g) — the config the headline metric is quoted on;
it fits one B200. Inputs are synthetic (include/ma_synth.h), generated on the
device; every step reads a gradient no earlier step saw (a shifted window of
one of up to 8 resident buffers); each step moves ~53 GB >> 126 MB L2, so no
L2 flush is needed between steps.

--impl reference times the reference's own CPU implementation
(oracle/_ref/libmicroadam_ref.so = the unmodified /root/reference sources) on
the host's cores: one MicroAdamOptimizer(blockwise=true) per thread over a
block-aligned shard of the same workload (bit-identical to the unsharded run),
value = Σ shard params / max per-thread step time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MicroAdam optimizer params/sec at 7B (1/2/4/8 B200); achieved HBM GB/s vs peak"
UNIT = "params/s"

WORKLOADS = {
    "llama2-7b": dict(dim=6_738_415_616, dtype="bf16",
                      desc="Llama-2-7B-sized flat vector (BASELINE configs[3])"),
    "llama2-13b": dict(dim=13_015_864_320, dtype="bf16",
                       desc="Llama-2-13B-sized flat vector (configs[4]; density / window sweep)"),
    "opt-1.3b": dict(dim=1_300_000_000, dtype="bf16", desc="OPT-1.3B-sized flat vector (configs[2])"),
    "bert-110m": dict(dim=110_000_000, dtype="f32", desc="BERT-base-sized flat vector (configs[1])"),
    "1m": dict(dim=1_000_000, dtype="f32", desc="synthetic 1M vector (configs[0])"),
}
DT_BYTES = {"f64": 8, "f32": 4, "bf16": 2}
MA_DT = {"f64": 0, "f32": 1, "bf16": 2}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="llama2-7b", choices=sorted(WORKLOADS))
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--window", type=int, default=10)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-shard-blocks", type=int, default=256)
    ap.add_argument("--mode", default="allgather", choices=["shard", "allgather", "sparse"],
                    help="N>1: 'allgather' (default, the north star's layout) = the workload's blocks "
                         "split across ranks, each step = the rank's shard step + the NCCL all-gather "
                         "of the updated bf16 θ shards into every rank's replica (ma_step_allgather's "
                         "two halves through the C ABI; strong scaling); 'sparse' = the workload split "
                         "across ranks for the EF / Top-K front, NCCL all-gather of the new window rows "
                         "only (ma_exchange_rows), ADAM_STATS + update replicated on every rank's θ "
                         "(strong scaling); 'shard' = each rank steps its own workload-sized block range "
                         "of an N x workload vector, no collective (weak scaling)")
    ap.add_argument("--grad-stream", default="normal", choices=["normal", "heavy"],
                    help="synthetic gradients: 'normal' (ma_synth Irwin-Hall(4)) or 'heavy' "
                         "(heavy-tailed, per-block scales: ma_synth_heavy)")
    return ap.parse_args()


# The gradient stream of the timed loop: step i (0-based, warm-up included)
# reads resident buffer i % n_grads — ma_synth stream step (i % n_grads) + 1 —
# at element offset off(i), so no step repeats an earlier gradient. Shared with
# tests/test_gpu_scale.py, which replays it against the oracle.
SHIFT = 64 * 4096
STEP8 = 1283  # offset step in units of 8 elements (16-byte aligned for bf16)


def grad_source(i: int, n_grads: int):
    """(ma_synth step, element offset) of the gradient bench step i reads."""
    return (i % n_grads) + 1, ((i // n_grads) * STEP8 * 8) % SHIFT


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# CPU reference timing (oracle/_ref = unmodified reference sources)
# ---------------------------------------------------------------------------
def host_cpu():
    """(model name, physical cores, logical CPUs) of this host (/proc/cpuinfo)."""
    model, cores = "unknown", set()
    phys = core = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                k, _, v = line.partition(":")
                k, v = k.strip(), v.strip()
                if k == "model name":
                    model = v
                elif k == "physical id":
                    phys = v
                elif k == "core id":
                    core = v
                elif not k and phys is not None:
                    cores.add((phys, core))
                    phys = core = None
        if phys is not None:
            cores.add((phys, core))
    except OSError:
        pass
    logical = os.cpu_count() or 1
    return model, (len(cores) or logical), logical


def cpu_reference_time(wl, args, steps, warmup, threads=None):
    """Time the reference's own step (oracle/_ref = the unmodified reference
    sources; the C restatement if the reference was not built) on this host:
    one MicroAdamOptimizer(blockwise=true) per thread over a block-aligned shard
    of the workload (bit-identical to the unsharded run),
    `warmup` untimed steps (at least m, so every timed step runs with a full
    window, like the GPU arm) then `steps` consecutive timed steps."""
    import numpy as np
    import oracle
    threads = threads or os.cpu_count() or 1
    shard = args.cpu_shard_blocks * 4096
    warmup = max(warmup, args.window)
    kind = "reference" if oracle.reference_available() else "port"
    if kind == "reference":
        L = oracle.ref_lib()
        per = np.zeros(threads)
        t = L.ref_time_shards(threads, shard, steps, warmup, MA_DT[wl["dtype"]], 4096, 64,
                              args.density, args.window, per)
        if t <= 0:
            raise RuntimeError("reference CPU timing failed")
    else:  # the C restatement, single thread (no reference build on this host)
        threads = 1
        o = oracle.Oracle(oracle.synth(1, 0, 0, shard, wl["dtype"]),
                          dict(density=args.density, window=args.window))
        for s in range(warmup):
            o.step(oracle.synth(42, s + 1, 0, shard, wl["dtype"]))
        t0 = time.perf_counter()
        for s in range(steps):
            o.step(oracle.synth(42, warmup + s + 1, 0, shard, wl["dtype"]))
        t = (time.perf_counter() - t0) / steps
    value = threads * shard / t
    model, phys, logical = host_cpu()
    sample = (f"{threads} threads on {model} ({phys} physical cores, {logical} logical CPUs); each thread "
              f"owns a {shard:,}-param block-aligned shard of the {wl['desc']} ({args.cpu_shard_blocks} "
              f"blocks of 4096) and runs {warmup} untimed steps (window full from step {args.window}) then "
              f"{steps} consecutive timed steps ({warmup + 1}..{warmup + steps}); value = "
              f"{threads}*{shard}/max over threads of mean s/step ({t:.4f} s)")
    return {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
            "s_per_step_per_thread": t, "cpu_model": model, "physical_cores": phys, "logical_cpus": logical}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    wl = WORKLOADS[args.workload]
    base = cpu_reference_time(wl, args, steps=args.steps, warmup=args.warmup)
    value = base["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, args.window), "warmup_requested": args.warmup,
        "ms_per_step": wl["dim"] / value * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (include/ma_synth.h stream, rounded to the workload dtype)",
        "config": {"workload": f"{args.workload}: {wl['desc']}, density {args.density}, "
                               f"m={args.window}, 4-bit EF, B_d=4096, B_q=64, blockwise",
                   "dim": wl["dim"], "sample": base["sample"],
                   "ms_per_step_note": "full-workload step time implied by the sampled shards' rate"},
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                               "physical_cores", "logical_cpus")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        sm = []
        mx = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for n, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def read_traffic(workload, dim):
    """DRAM bytes per launch from the committed ncu capture (profiles/), scaled per param."""
    p = os.path.join(ROOT, "profiles", "ncu_step_kernel.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d["dram_bytes_per_param"] * dim, d.get("source")
    except Exception:
        return None, None


def algorithmic_bytes(lay, gdt, pdt, vdt, m):
    """Bytes one step must move: g read, θ read+write, EF codes and
    (lo, hi) read+write, one window row written + (m-1) rows read."""
    d = lay.dim
    return (d * DT_BYTES[gdt] + 2 * d * DT_BYTES[pdt] + 2 * lay.code_bytes + 2 * 16 * lay.num_buckets
            + m * lay.row_width * (2 + DT_BYTES[vdt]))


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2405_15593_b200 as ma
    from paper_2405_15593_b200 import sharding

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = WORKLOADS[args.workload]
    d, dt = wl["dim"], wl["dtype"]
    gdt = pdt = dt
    vdt = "bf16"
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[dt]
    hp = ma.HyperParams(density=args.density, window=args.window, lr=1e-3)
    # BENCH_FORCE_COMM=1: run the N>1 collective code path with a 1-rank NCCL
    # communicator (a smoke test of the multi-GPU layout on a one-GPU box)
    force_comm = os.environ.get("BENCH_FORCE_COMM") == "1"
    gather = (world > 1 or force_comm) and args.mode == "allgather"
    sparse = args.mode == "sparse"
    levels = 2 if args.grad_stream == "heavy" else 0
    comm = None
    if (world > 1 or force_comm) and args.mode in ("allgather", "sparse"):
        # the library's own NCCL communicator (ma_comm_init); torch.distributed only
        # carries the 128-byte unique id and the timing reductions
        uid = [ma.Comm.unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        comm = ma.Comm(uid[0], world, rank, local)
    if sparse:  # strong scaling, window-row exchange: a whole-vector handle per rank
        if d % hp.block:
            raise SystemExit("--mode sparse needs a whole-block workload")
        dim_total = d
        b0, b1, e0, e1 = sharding.partition_blocks(d, hp.block, world, rank)
        stride = sharding.shard_stride(d, hp.block, world)
    elif gather:  # strong scaling: the workload's blocks split over the ranks
        dim_total = d
        b0, b1, e0, e1 = sharding.partition_blocks(d, hp.block, world, rank)
        stride = sharding.shard_stride(d, hp.block, world)
    else:  # weak scaling: rank r owns ~1/N of the blocks of a world x d vector
        dim_total = d * world
        b0, b1, e0, e1 = sharding.partition_blocks(dim_total, hp.block, world, rank)
    n = e1 - e0
    eng = ma.MicroAdam(dim_total, hp, param_dtype=pdt, grad_dtype=gdt, value_dtype=vdt,
                       block_range=(0, -1) if sparse else (b0, b1), device=local)
    lay = eng.layout
    lib = ma.lib()
    stream = torch.cuda.current_stream()

    def fill(t, seed, step, offset, count):
        ma._capi.check(lib.ma_fill_synthetic(t.data_ptr(), MA_DT[dt], count, seed, step, offset,
                                             levels if seed == 42 else 0, stream.cuda_stream))

    if sparse:  # every rank holds the full θ replica; rows travel, θ does not
        full = None
        params = torch.empty(d, dtype=tdt, device="cuda")
        sblk = stride // hp.block  # blocks per rank (padded)
        stage = eng.stage_buffers(sblk)
        rows = eng.stage_buffers(sblk * world)
    elif gather:
        full = torch.empty(stride * world, dtype=tdt, device="cuda")
        params = full[rank * stride: rank * stride + n]
    else:
        full = None
        params = torch.empty(n, dtype=tdt, device="cuda")
    fill(params, 1, 0, 0 if sparse else e0, params.numel())
    # Every step gets a gradient no earlier step saw: up to 8 resident buffers
    # (as many as HBM allows, >= 2), each SHIFT elements longer than the shard,
    # and step i reads buffer i % B at offset (i // B) * STEP8 * 8 elements.
    # Re-feeding an identical gradient every B steps (B < m) would make the
    # window and the EF see exact repeats, which real training never produces.
    free, _ = torch.cuda.mem_get_info()
    gbytes = (n + SHIFT) * DT_BYTES[gdt]
    reserve = 2 * n * DT_BYTES[gdt] + (8 << 30)  # e2e staging (θ + g copies) + headroom
    n_grads = int(max(2, min(8, args.steps + args.warmup, (free - reserve) // gbytes)))
    grads = [torch.empty(n + SHIFT, dtype=tdt, device="cuda") for _ in range(n_grads)]
    for i, g in enumerate(grads):
        fill(g, 42, i + 1, e0, n + SHIFT)
    torch.cuda.synchronize()

    def grad_view(i):
        j, off = grad_source(i, n_grads)
        return grads[j - 1][off: off + n]

    nb_all = d // hp.block

    def one_step(i, ev=None):
        # ev = (start, after the step kernel(s), after the collective)
        if ev is not None:
            ev[0].record()
        if sparse:
            eng.step_front(grad_view(i), b0, b1, stage, stream=stream.cuda_stream)
            if ev is not None:
                ev[1].record()
            if comm is not None:
                eng.exchange_rows(stage, rows, comm, stream=stream.cuda_stream)  # ma_exchange_rows
            if ev is not None:
                ev[2].record()
            eng.step_stats(params, 1e-3, stream=stream.cuda_stream)
        else:
            # ma_step_allgather = this step + ma_allgather_params; called as its two
            # halves so the collective is timed on its own
            eng.step(params, grad_view(i), 1e-3, stream=stream.cuda_stream)
            if ev is not None:
                ev[1].record()
            if gather:
                eng.allgather_params(full, comm, stream=stream.cuda_stream)
            if ev is not None:
                ev[2].record()

    # untimed warm-up: at least m steps, so every timed step runs with a full
    # window (filled = m) like a training run past its first m steps
    warm = max(args.warmup, args.window)
    for i in range(warm):
        one_step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = eng.kernel_launches()
    kev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0.record()
    for i in range(args.steps):
        one_step(warm + i, kev[i])
    t1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = eng.kernel_launches() - launches0
    eng.synchronize()
    elapsed = t0.elapsed_time(t1) / 1e3
    coll = sum(b.elapsed_time(c) for a, b, c in kev) / 1e3 / args.steps
    if sparse:  # front + stats kernels: the step minus the row exchange
        kern = elapsed / args.steps - coll
    else:
        kern = sum(a.elapsed_time(b) for a, b, c in kev) / 1e3 / args.steps
    if world > 1:
        tt = torch.tensor([elapsed, kern, coll], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed, kern, coll = float(tt[0]), float(tt[1]), float(tt[2])
    s_per_step = elapsed / args.steps
    value = dim_total / s_per_step

    peak, peak_src = read_peaks()
    bytes_launch = algorithmic_bytes(lay, gdt, pdt, vdt, hp.window)
    achieved = bytes_launch / kern / 1e9
    traffic_total, traffic_src = read_traffic(args.workload, n)

    # ---- end to end through the reference-facing host path (ma_step_host) ----
    e2e = None
    if not args.no_e2e and not (sparse and world > 1):
        h_params = torch.empty(n, dtype=tdt, pin_memory=True)
        h_grads = [torch.empty(n, dtype=tdt, pin_memory=True) for _ in range(2)]
        h_params.copy_(params)
        for k, hg in enumerate(h_grads):
            hg.copy_(grad_view(k))
        del grads
        torch.cuda.empty_cache()
        eng.set_params(h_params)
        eng.step_host(h_params, h_grads[0], 1e-3)  # warm-up (allocates staging)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        for i in range(args.e2e_steps):
            eng.step_host(h_params, h_grads[(i + 1) % 2], 1e-3)
        te = (time.perf_counter() - t) / args.e2e_steps
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        # the PCIe floor: the same gradient bytes copied H2D alone (pinned, one stream)
        dg = torch.empty(n, dtype=tdt, device="cuda")
        dg.copy_(h_grads[0], non_blocking=True)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        dg.copy_(h_grads[1], non_blocking=True)
        ev1.record()
        torch.cuda.synchronize()
        h2d_ms = ev0.elapsed_time(ev1)
        # and both directions at once (g up, θ down on a second stream): the
        # full-duplex floor the chunked ma_step_host pipeline can approach
        dth = torch.empty(n, dtype=tdt, device="cuda")
        side = torch.cuda.Stream()
        torch.cuda.synchronize()
        t_dx = time.perf_counter()
        with torch.cuda.stream(side):
            h_params.copy_(dth, non_blocking=True)
        dg.copy_(h_grads[0], non_blocking=True)
        torch.cuda.synchronize()
        duplex_ms = (time.perf_counter() - t_dx) * 1e3
        del dg, dth
        eng.set_params(h_params)  # h_params was overwritten by the probe
        lay = eng.layout
        if os.environ.get("MA_HOST_SPARSE") == "1":
            # window ring indices (int16) + θ gathered at them, scattered on host threads
            d2h = lay.num_blocks * args.window * lay.kb_stride * (2 + DT_BYTES[pdt])
            ret = "θ at the window coordinates D2H (ring idx + gathered θ), host-thread scatter"
        else:
            d2h, ret = n * DT_BYTES[pdt], "updated θ D2H (dense)"
        e2e = {"value": dim_total / te, "unit": UNIT, "h2d_bytes_per_step": n * DT_BYTES[gdt],
               "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "ms_per_step": te * 1e3, "h2d_only_ms": h2d_ms, "h2d_plus_d2h_concurrent_ms": duplex_ms,
               "h2d_only_gbs": n * DT_BYTES[gdt] / h2d_ms / 1e6,
               "path": "ma_step_host (C ABI): pinned host g -> H2D, fused step, " + ret + ", "
                       "chunked so copies overlap the kernel; host wall clock around the "
                       "synchronous call"}
        del h_params, h_grads

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_reference_time(wl, args, steps=3, warmup=args.window)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                      "physical_cores", "logical_cpus")}
        except Exception as exc:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": warm, "warmup_requested": args.warmup,
            "ms_per_step": s_per_step * 1e3,
            "higher_is_better": True, "scaling": "strong" if (gather or sparse) else "weak",
            "vs_baseline": None,
            "dtype": dt,
            "data": f"synthetic (include/ma_synth.h " + (
                "heavy-tailed per-block-scaled stream" if levels == 2 else "Irwin-Hall(4) stream") +
                    f", generated on device; step i reads a shifted window of resident buffer i % "
                    f"{n_grads}, so no step repeats a gradient; {warm} untimed steps first, so every "
                    f"timed step runs with a full window)",
            "config": {
                "workload": f"{args.workload}: {wl['desc']}, {d:,} params, {dt} θ/g, bf16 window "
                            f"values, density {args.density}, m={args.window}, 4-bit EF, "
                            f"B_d=4096, B_q=64, blockwise Top-K",
                "dim": d, "dim_total": dim_total,
                "parallelism": f"block-sharded dp{world}" + (
                    " + NCCL all-gather of the updated bf16 θ shards each step (ma_allgather_params)"
                    if gather else
                    (" EF/Top-K front + NCCL all-gather of the new window rows (ma_exchange_rows), "
                     "ADAM_STATS + update replicated on each rank's θ" if sparse else None) or
                    (", one workload-sized block range per rank, no data-path collective"
                     if world > 1 else "")),
                "l2": "no flush: every step streams ~%.0f GB >> 126 MB L2" % (
                    bytes_launch * world / 1e9),
                "grad_buffers": n_grads},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": (traffic_total if traffic_total is None else traffic_total),
                         "algorithmic_bytes_per_launch": bytes_launch,
                         "bytes_per_param": bytes_launch / n,
                         "kernel_ms": kern * 1e3,
                         "kernel_ms_per_step": [round(a.elapsed_time(b_), 3) for a, b_, _ in kev],
                         "peak_source": peak_src,
                         "traffic_source": traffic_src,
                         "kernel": "microadam_step_lean (one warp per B_d=4096 Top-K block: fp32-screened EF "
                                   "decode + Top-K, window row, exact fp64 4-bit re-quantization, "
                                   "ADAM_STATS + θ update)"},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clk,
        }
        if gather or (sparse and comm is not None):
            psz = DT_BYTES[pdt]
            recv = ((world - 1) * stride * psz if gather else
                    (world - 1) * (stride // hp.block) * lay.kb_stride * (2 + DT_BYTES[vdt]))
            line["step_only"] = {"value": d / kern, "ms": kern * 1e3}
            line["collective"] = {
                "op": ("ncclAllGather of the bf16 θ shards (ma_allgather_params)" if gather else
                       "ncclAllGather of the new window rows (ma_exchange_rows)"),
                "ms": coll * 1e3, "bytes_received_per_rank": recv,
                "algbw_gbs": recv / coll / 1e9 if coll > 0 else None,
                "timing": "CUDA events around the collective on the step stream, mean over the timed "
                          "steps, max over ranks"}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
