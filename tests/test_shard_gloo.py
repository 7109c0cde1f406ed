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


def _he_worker(rank, world_size, port, q, on_gpu):
    """One rank of a sharded batched run: its own context and session
    (keys replicated from the shared seed), its own disjoint image range,
    decrypted logits checked against forward_integer; only the mismatch
    count and the timing cross ranks (sum / max over gloo)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        from oracle import refbind as R

        per = 3
        rng = shard_range(per * world_size, world_size, rank)
        net = nets.toy_net()
        imgs = nets.images(9, net, len(rng), start=rng.start)
        want = [R.forward_integer(net, x) for x in imgs]
        if on_gpu:
            import torch

            from paper_1812_10659_b200.bfv import BfvContext
            from paper_1812_10659_b200.lola import Session
            from paper_1812_10659_b200.params import make_params

            torch.cuda.set_device(0)
            cx = BfvContext(make_params(4096, L=7, T=3, K=1, seed=5))
            sess = Session(cx, net, "lola-mnist", len(rng))
            got, _, _ = sess.run(imgs)
        else:
            # the reference ring backend on the rank (plaintext semantics)
            from paper_1812_10659_b200.params import plain_primes

            rs = R.RefSession(net, "lola-mnist", 4096, plain_primes(4096, 3))
            got = [rs.run(x, decode=True)[0] for x in imgs]
        bad = sum(int(g != w) for g, w in zip(got, want))
        total_bad = sum_over_ranks(float(bad), world_size, device="cpu")
        total = sum_over_ranks(float(len(rng)), world_size, device="cpu")
        q.put((rank, list(rng), bad, total_bad, total))
    finally:
        dist.destroy_process_group()


def run_he_ranks(on_gpu: bool):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_he_worker, args=(r, 2, port, q, on_gpu)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (_, idx0, b0, tb0, n0), (_, idx1, b1, tb1, n1) = res
    assert set(idx0).isdisjoint(idx1) and sorted(idx0 + idx1) == list(range(6))
    assert b0 == b1 == 0 and tb0 == tb1 == 0.0 and n0 == n1 == 6.0


def test_two_rank_he_on_cpu_ranks():
    """Each rank runs inference over its shard (reference ring backend on
    CPU) and the mismatch count is summed across ranks."""
    run_he_ranks(on_gpu=False)


@pytest.mark.gpu
def test_two_rank_he_on_gpu_ranks():
    """Two ranks on cuda:0, each with its own BFV context and session over a
    disjoint image range; every rank's decrypted logits == forward_integer.
    (Independent ranks: no kernel of one waits on the other.)"""
    run_he_ranks(on_gpu=True)
