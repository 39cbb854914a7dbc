"""Data-parallel collectives behind the C ABI: ma_comm_*,
ma_step_allgather, ma_allgather_params, ma_exchange_rows.

The pool has one GPU per box and NCCL refuses two ranks on one device, so:
* the NCCL entry points run with a 1-rank communicator made through the ABI
  (ncclGetUniqueId / ncclCommInitRank loaded at run time) and must equal the
  plain step bit for bit — this exercises the library's NCCL loading, the
  partition checks and the in-place all-gather / broadcast code paths;
* the multi-rank data plane runs as 2 processes on cuda:0, each owning the
  library shard handle of its rank (ma_create_shard over sharding.py's block
  range), exchanging the updated θ shards through torch.distributed / gloo the
  way ma_step_allgather exchanges them over NVLink, and is compared bit for bit
  with the unsharded oracle run (compress.cpp:73-85: the Top-K partitions by
  block; window.cpp:43: the bias correction uses the replicated global step).
"""
import os
import socket

import numpy as np
import pytest

import oracle
from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

BLK = 4096


def _dev(x, dt="bf16"):
    import torch
    t = {"bf16": torch.bfloat16, "f32": torch.float32}[dt]
    return torch.from_numpy(np.ascontiguousarray(x, np.float64)).to(t).cuda()


def _comm1():
    from paper_2405_15593_b200 import Comm
    return Comm(Comm.unique_id(), 1, 0, 0)


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_step_allgather_one_rank_equals_step(dt):
    import torch
    from paper_2405_15593_b200 import MicroAdam
    d, hp = BLK * 30 + 777, dict(lr=1e-2, window=5)
    comm = _comm1()
    a = MicroAdam(d, hp, param_dtype=dt, grad_dtype=dt, value_dtype="bf16")
    b = MicroAdam(d, hp, param_dtype=dt, grad_dtype=dt, value_dtype="bf16", block_range=(0, -1))
    th0 = oracle.synth(1, 0, 0, d, dt)
    pa, pb = _dev(th0, dt), _dev(th0, dt)
    for s in range(1, 9):
        g = _dev(oracle.synth(42, s, 0, d, dt), dt)
        a.step(pa, g, 1e-2)
        rep = b.step_allgather(pb, g, comm, 1e-2, report=(s == 8))
    torch.cuda.synchronize()
    assert torch.equal(pa, pb)
    assert np.array_equal(a.error_buffer().codes, b.error_buffer().codes)
    assert rep is not None and rep.update_nnz > 0
    comm.close()


def test_allgather_rejects_a_foreign_partition():
    import torch
    from paper_2405_15593_b200 import InvalidArgument, MicroAdam
    d = BLK * 8
    comm = _comm1()
    eng = MicroAdam(d, dict(), param_dtype="bf16", grad_dtype="bf16", block_range=(0, 4))  # half the blocks
    p = torch.zeros(d, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(InvalidArgument):
        eng.allgather_params(p, comm)
    comm.close()


def test_exchange_rows_one_rank_equals_fused_step():
    import torch
    from paper_2405_15593_b200 import MicroAdam
    d, hp = BLK * 16, dict(lr=1e-2, window=4)
    comm = _comm1()
    fused = MicroAdam(d, hp, param_dtype="bf16", grad_dtype="bf16")
    split = MicroAdam(d, hp, param_dtype="bf16", grad_dtype="bf16")
    th0 = oracle.synth(1, 0, 0, d)
    pf, ps = _dev(th0), _dev(th0)
    nb = d // BLK
    stage, rows = split.stage_buffers(nb), split.stage_buffers(nb)
    for s in range(1, 8):
        g = _dev(oracle.synth(42, s, 0, d))
        fused.step(pf, g, 1e-2)
        split.step_front(g, 0, nb, stage)
        split.exchange_rows(stage, rows, comm)
        split.step_stats(ps, 1e-2)
    torch.cuda.synchronize()
    assert torch.equal(pf, ps)
    comm.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, d, steps, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2405_15593_b200 import MicroAdam, sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    hp = dict(lr=1e-2, window=4)
    b0, b1, e0, e1 = sharding.partition_blocks(d, BLK, world, rank)
    stride = sharding.shard_stride(d, BLK, world)
    eng = MicroAdam(d, hp, param_dtype="bf16", grad_dtype="bf16", block_range=(b0, b1))
    full = _dev(oracle.synth(1, 0, 0, d, "bf16"))  # every rank's θ replica
    for s in range(1, steps + 1):
        g = _dev(oracle.synth(42, s, e0, e1 - e0, "bf16"))  # only this rank's gradient shard
        eng.step(full[e0:e1], g, 1e-2)
        # the all-gather of the updated shards (ma_step_allgather's exchange), staged through gloo
        mine = torch.zeros(2 * stride, dtype=torch.uint8)  # bf16 bytes (gloo has no 16-bit ints)
        mine[: 2 * (e1 - e0)] = full[e0:e1].view(torch.uint8).cpu()
        parts = [torch.empty(2 * stride, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(parts, mine)
        full.copy_(torch.cat(parts)[: 2 * d].view(torch.bfloat16).cuda())
    torch.cuda.synchronize()
    eb = eng.error_buffer()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), theta=full.view(torch.int16).cpu().numpy(),
             codes=eb.codes, lo=eb.lo, hi=eb.hi, e0=e0, e1=e1)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("d,world", [(BLK * 13 + 300, 2)])
def test_two_process_shards_match_unsharded_oracle(d, world, tmp_path):
    import torch.multiprocessing as mp
    steps = 6
    mp.start_processes(_rank_main, args=(world, _free_port(), d, steps, str(tmp_path)), nprocs=world,
                       start_method="spawn")
    orc = oracle.Oracle(oracle.synth(1, 0, 0, d, "bf16"), dict(lr=1e-2, window=4), param_dtype="bf16",
                        value_dtype="bf16")
    for s in range(1, steps + 1):
        orc.step(oracle.synth(42, s, 0, d, "bf16"), 1e-2)
    st = orc.state()
    want = st.params.astype(np.float32).view(np.uint32) >> 16
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        theta = z["theta"].view(np.uint16).astype(np.uint32)
        assert np.array_equal(theta, want), f"rank {r}: θ replica differs from the unsharded oracle"
        e0, e1 = int(z["e0"]), int(z["e1"])
        assert np.array_equal(z["codes"], st.codes[e0 // 2: (e1 + 1) // 2]), f"rank {r}: EF codes differ"
        assert np.array_equal(z["lo"].view(np.uint64), st.lo[e0 // 64: (e1 + 63) // 64].view(np.uint64))
