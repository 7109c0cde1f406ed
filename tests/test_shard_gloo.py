"""Multi-rank path on CPU: world_size 2 over gloo. Shards are disjoint and
cover the job, timing is the max over ranks, the image count the sum."""
from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1812_10659_b200 import nets
from paper_1812_10659_b200.shard import max_over_ranks, shard_range, sum_over_ranks


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world_size, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        per = 3
        rng = shard_range(per * world_size, world_size, rank)
        net = nets.toy_net()
        imgs = nets.images(2, net, len(rng), start=rng.start)
        elapsed = 1.0 + rank  # stand-in for the device-timed seconds
        t = max_over_ranks(elapsed, world_size, device="cpu")
        n = sum_over_ranks(float(len(rng)), world_size, device="cpu")
        q.put((rank, list(rng), imgs.sum(), t, n))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_and_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, idx0, s0, t0, n0), (r1, idx1, s1, t1, n1) = res
    assert set(idx0).isdisjoint(idx1) and sorted(idx0 + idx1) == list(range(6))
    assert t0 == t1 == 2.0 and n0 == n1 == 6.0
    # a rank's images are exactly the global set's slice
    net = nets.toy_net()
    assert s0 == nets.images(2, net, 3, start=0).sum() and s1 == nets.images(2, net, 3, start=3).sum()


def test_shard_range_edges():
    assert list(shard_range(0, 4, 2)) == []
    assert [len(shard_range(10, 3, r)) for r in range(3)] == [3, 3, 4]
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
