"""Batch sharding on CPU: the partition, and the two
out-of-band collectives (max of per-rank device time, verification gather)
exercised with world_size 2 over gloo."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2601_11608_b200 import shard


@pytest.mark.parametrize("n,world", [(8192, 1), (8192, 2), (8192, 8), (7, 3), (3, 8), (0, 2), (1000003, 8)])
def test_shard_range_partitions_the_batch(n, world):
    spans = [shard.shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, _) in zip(spans, spans[1:]):
        assert b == c  # contiguous, no gap, no overlap
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1 and sum(sizes) == n


def test_shard_range_rejects_bad_ranks():
    for rank, world in ((0, 0), (2, 2), (-1, 4)):
        with pytest.raises(ValueError):
            shard.shard_range(16, rank, world)


def test_single_process_collectives_are_identity():
    assert shard.max_over_ranks(3.5) == 3.5
    assert shard.gather_scalars([1.0, 2.0]) == [[1.0, 2.0]]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist
    r, local, w = shard.dist_env()
    shard.init("gloo")
    try:
        lo, hi = shard.shard_range(8192, r, w)
        ms = 10.0 + r  # per-rank "device time"
        mx = shard.max_over_ranks(ms)
        got = shard.gather_scalars([float(lo), float(hi), ms])
        # unequal shards (7 images over 2 ranks) collected on rank 0
        a, b = shard.shard_range(7, r, w)
        mine = torch.arange(a, b, dtype=torch.float32).reshape(-1, 1).repeat(1, 3)
        full = shard.gather_to(mine, [y - x for x, y in (shard.shard_range(7, k, w) for k in range(w))], dst=0)
        q.put((r, local, w, lo, hi, mx, got, None if full is None else full.tolist()))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_two_rank_gloo_shard_and_reduce():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spans = [(lo, hi) for (_, _, _, lo, hi, _, _, _) in res]
    assert spans == [(0, 4096), (4096, 8192)]
    for (r, local, w, _, _, mx, got, full) in res:
        assert w == 2 and local == r
        assert mx == 11.0
        if r == 0:
            assert full == [[float(i)] * 3 for i in range(7)]
        else:
            assert full is None  # max over ranks, as bench.py times multi-GPU runs
        assert got == [[0.0, 4096.0, 10.0], [4096.0, 8192.0, 11.0]]


def _gather_worker(rank, world, port, dst, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist
    shard.init("gloo")
    try:
        sizes = [b - a for a, b in (shard.shard_range(n, k, world) for k in range(world))]
        a, b = shard.shard_range(n, rank, world)
        mine = torch.arange(a * 6, b * 6, dtype=torch.float32).reshape(-1, 2, 3)
        full = shard.gather_to(mine, sizes, dst=dst)
        bad = None
        try:
            shard.gather_to(mine[:0] if sizes[rank] else torch.zeros(1, 2, 3), sizes, dst=dst)
        except ValueError as e:
            bad = str(e)
        # a mismatch on ONE rank only: every rank raises (nobody is left blocked in irecv)
        one_bad = False
        try:
            shard.gather_to(torch.zeros(sizes[0] + 1, 2, 3) if rank == 0 else mine, sizes, dst=dst)
        except ValueError:
            one_bad = True
        q.put((rank, None if full is None else full.tolist(), bad is not None and one_bad))
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dst,n", [(3, 1, 7), (4, 3, 2)])
def test_gather_to_lands_only_on_dst(world, dst, n):
    """gather_to: point-to-point sends into dst's slices (unequal and empty shards, dst != 0);
    the other ranks receive nothing; a shard that does not match its size is rejected."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, dst, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = torch.arange(n * 6, dtype=torch.float32).reshape(n, 2, 3).tolist()
    for r, full, rejected in res:
        assert full == (want if r == dst else None)
        assert rejected
