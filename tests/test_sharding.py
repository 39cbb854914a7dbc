"""Block-aligned data-parallel sharding — CPU tests.

* the partition covers every block exactly once, contiguously, with the
  padded-chunk layout bench.py all-gathers;
* block-aligned shards of the oracle step reproduce the unsharded step
  bit-for-bit (the property the device shards rely on);
* world_size 2 over torch.distributed / gloo: each rank steps its shard and one
  all_gather_into_tensor of padded shards rebuilds θ identical to the
  unsharded run (the multi-GPU host logic of bench.py, minus the GPU).
"""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2405_15593_b200 import sharding


def test_partition_covers_blocks_exactly():
    for dim, block, world in [(6_738_415_616, 4096, 8), (1_000_000, 4096, 3), (100_003, 4096, 2),
                              (4096 * 5, 4096, 5), (37, 8, 2)]:
        nb = sharding.num_blocks(dim, block)
        prev = 0
        stride = sharding.shard_stride(dim, block, world)
        for r in range(world):
            b0, b1, e0, e1 = sharding.partition_blocks(dim, block, world, r)
            assert b0 == prev and b1 > b0
            assert e0 == b0 * min(block, dim) and e1 == min(b1 * min(block, dim), dim)
            assert e1 - e0 <= stride and e0 == r * stride
            prev = b1
        assert prev == nb
        assert sum(sharding.shard_sizes(dim, block, world)) == dim


def test_llama7b_partition_counts():
    counts = [b1 - b0 for b0, b1, _, _ in
              (sharding.partition_blocks(6_738_415_616, 4096, 8, r) for r in range(8))]
    assert counts[:7] == [205_641] * 7 and counts[7] == 1_645_121 - 7 * 205_641


def test_partition_rejects_empty_ranks():
    with pytest.raises(ValueError):
        sharding.partition_blocks(4096 * 3, 4096, 5, 4)


def _shard_run(theta0, grads, hp, dim, world, rank):
    b0, b1, e0, e1 = sharding.partition_blocks(dim, hp["block"], world, rank)
    o = oracle.Oracle(theta0[e0:e1], hp)
    for g in grads:
        o.step(g[e0:e1])
    return o.state(), e0, e1


@pytest.mark.parametrize("dim,world", [(4096 * 6 + 1000, 2), (4096 * 9 + 17, 3)])
def test_oracle_shards_are_bit_identical(dim, world):
    hp = dict(block=4096, bucket=64, window=4, lr=1e-2)
    theta0 = oracle.synth(1, 0, 0, dim)
    grads = [oracle.synth(42, s, 0, dim, "f32") for s in range(1, 7)]
    full = oracle.Oracle(theta0, hp)
    for g in grads:
        full.step(g)
    sf = full.state()
    params = np.concatenate([_shard_run(theta0, grads, hp, dim, world, r)[0].params
                             for r in range(world)])
    codes = np.concatenate([_shard_run(theta0, grads, hp, dim, world, r)[0].codes
                            for r in range(world)])
    assert np.array_equal(params.view(np.uint64), sf.params.view(np.uint64))
    assert np.array_equal(codes, sf.codes)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, dim, out_path):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hp = dict(block=4096, bucket=64, window=3, lr=1e-2)
    theta0 = oracle.synth(1, 0, 0, dim)
    grads = [oracle.synth(42, s, 0, dim, "f32") for s in range(1, 5)]
    st, e0, e1 = _shard_run(theta0, grads, hp, dim, world, rank)
    stride = sharding.shard_stride(dim, hp["block"], world)
    mine = torch.zeros(stride, dtype=torch.float64)
    mine[: e1 - e0] = torch.from_numpy(st.params)
    full = torch.empty(stride * world, dtype=torch.float64)
    dist.all_gather_into_tensor(full, mine)
    if rank == 0:
        np.save(out_path, full[:dim].numpy())
    dist.destroy_process_group()


def test_gloo_world2_allgather_rebuilds_unsharded_params(tmp_path):
    import torch.multiprocessing as mp
    dim, world = 4096 * 5 + 333, 2
    out = str(tmp_path / "theta.npy")
    mp.spawn(_gloo_worker, args=(world, _free_port(), dim, out), nprocs=world, join=True)
    hp = dict(block=4096, bucket=64, window=3, lr=1e-2)
    full = oracle.Oracle(oracle.synth(1, 0, 0, dim), hp)
    for s in range(1, 5):
        full.step(oracle.synth(42, s, 0, dim, "f32"))
    got = np.load(out)
    assert np.array_equal(got.view(np.uint64), full.state().params.view(np.uint64))
