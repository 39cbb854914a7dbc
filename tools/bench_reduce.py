"""Fused gradient reduce-scatter + step (ma_step_reduce) vs reduce-then-step.

One process per GPU. Under torchrun (WORLD_SIZE > 1) every rank allocates its
full gradient in torch symmetric memory and steps its block shard reading the
shard range from every rank's buffer over NVLink (peer pointers). On one GPU
(the default) it emulates rank 0 of an N-rank job: the shard of the workload
that rank would own, with the N ranks' gradients as local HBM buffers.

Prints one JSON line per variant: fused (lean kernel reads the sources block by
block), unfused (reduce kernel into the gradient buffer, then the step) and
torch (fp32 torch sum + cast, then the step). Device time per step, CUDA events.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2405_15593_b200 as ma  # noqa: E402
from paper_2405_15593_b200 import sharding  # noqa: E402

DIMS = {"llama2-7b": 6_738_415_616, "opt-1.3b": 1_315_758_080}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama2-7b", choices=sorted(DIMS))
    ap.add_argument("--ranks", type=int, default=8, help="emulated ranks on one GPU")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    nr = world if world > 1 else args.ranks
    d = DIMS[args.workload]
    b0, b1, e0, e1 = sharding.partition_blocks(d, 4096, nr, rank)
    n = e1 - e0
    hp = ma.HyperParams(lr=1e-3)
    lib = ma.lib()
    stream = torch.cuda.current_stream()
    SHIFT = 64 * 4096
    nbuf = 2

    def fill(t, seed, step, offset):
        ma._capi.check(lib.ma_fill_synthetic(t.data_ptr(), 2, t.numel(), seed, step, offset, 0,
                                             stream.cuda_stream))

    if world > 1:
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        bufs, ptrs = [], []
        for k in range(nbuf):
            t = symm.empty(d + SHIFT, dtype=torch.bfloat16, device="cuda")
            fill(t, 42 + rank, k + 1, 0)
            h = symm.rendezvous(t, dist.group.WORLD)
            bufs.append((t, h))
            ptrs.append(list(h.buffer_ptrs))
        torch.cuda.synchronize()
        dist.barrier()

        def sources(i):
            k = i % nbuf
            off = ((i // nbuf) * 1283 * 8) % SHIFT
            return [p + (off + e0) * 2 for p in ptrs[k]]
    else:
        bufs = [[torch.empty(n + SHIFT, dtype=torch.bfloat16, device="cuda") for _ in range(nr)]
                for _ in range(nbuf)]
        for k in range(nbuf):
            for r in range(nr):
                fill(bufs[k][r], 42 + r, k + 1, e0)

        def sources(i):
            k = i % nbuf
            off = ((i // nbuf) * 1283 * 8) % SHIFT
            return [b[off: off + n] for b in bufs[k]]

    scale = 1.0 / nr
    out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    sc = torch.tensor(scale, dtype=torch.float32, device="cuda")

    def run(variant):
        eng = ma.MicroAdam(d, hp, param_dtype="bf16", grad_dtype="bf16", value_dtype="bf16",
                           block_range=(b0, b1), device=local)
        params = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        fill(params, 1, 0, e0)
        os.environ.pop("MA_RS_UNFUSED", None)
        if variant == "unfused":
            os.environ["MA_RS_UNFUSED"] = "1"

        def step(i):
            srcs = sources(i)
            if world > 1:
                bufs[i % nbuf][1].barrier(channel=0)
            if variant == "torch":
                acc = srcs[0].float() if not isinstance(srcs[0], int) else None
                for s in srcs[1:]:
                    acc = acc + s.float()
                out.copy_((acc * sc).to(torch.bfloat16))
                eng.step(params, out, 1e-3, stream=stream.cuda_stream)
            else:
                eng.step_reduce(params, out, srcs, scale, 1e-3, stream=stream.cuda_stream)

        for i in range(args.warmup):
            step(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for i in range(args.steps):
            step(args.warmup + i)
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / args.steps
        if world > 1:
            tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt[0])
        os.environ.pop("MA_RS_UNFUSED", None)
        del eng, params
        torch.cuda.empty_cache()
        return ms

    for variant in (["fused", "unfused"] if world > 1 else ["fused", "unfused", "torch"]):
        ms = run(variant)
        if rank == 0:
            src_bytes = nr * n * 2
            print(json.dumps({
                "variant": variant, "workload": args.workload, "ranks": nr, "real_ranks": world,
                "shard_params": n, "ms_per_step": ms, "shard_params_per_s": n / ms * 1e3,
                "job_params_per_s": d / ms * 1e3 if world > 1 else None,
                "source_GBps": src_bytes / ms / 1e6,
                "sources": "peer (symmetric memory, NVLink)" if world > 1 else "local HBM buffers"}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
