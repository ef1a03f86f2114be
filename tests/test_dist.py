"""Multi-rank host logic on CPU (gloo, world_size 2): request sharding,
max-over-ranks timing, and the post-run gather. The GPU path
uses the same functions over NCCL; nothing here needs a GPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_08314_b200 import replicas


def test_shard_partitions_requests():
    for n in (0, 1, 7, 256, 257):
        for world in (1, 2, 4, 8):
            got = [replicas.shard(n, world, r) for r in range(world)]
            flat = [i for g in got for i in g]
            assert flat == list(range(n))
            sizes = [len(g) for g in got]
            assert max(sizes) - min(sizes) <= 1
    assert replicas.shard(256, 8, 3) == range(96, 128)
    with pytest.raises(ValueError):
        replicas.shard(4, 2, 2)


def test_waves():
    w = replicas.waves(range(10, 75), 32)
    assert [len(x) for x in w] == [32, 32, 1]
    assert w[0].start == 10 and w[-1].stop == 75


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 5
        mine = replicas.shard(n, world, rank)
        # each "request" generates 3 tokens: id*10 + step
        rows = torch.tensor([[i * 10 + s for s in range(3)] for i in mine], dtype=torch.int32).reshape(-1, 3)
        allr = replicas.gather_rows(dist, rows, n)
        replicas.barrier(dist)
        t = replicas.max_over_ranks(dist, 1.5 + rank)
        s = replicas.sum_over_ranks(dist, float(len(mine)))
        q.put((rank, allr.tolist(), t, s))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_timing():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, rows, t, s in res:
        assert rows == [[i * 10 + k for k in range(3)] for i in range(5)]
        assert t == 2.5  # max over ranks
        assert s == 5.0


class _StubSession:
    """Deterministic stand-in for a batched Session: token j of a request is a
    function of its prompt only, so the gathered table is layout-independent."""

    def __init__(self, batch):
        self.batch = batch

    def reset(self):
        pass

    def generate(self, prompts, gen):
        import numpy as np

        assert prompts.shape[0] == self.batch
        base = prompts.astype(np.int64).sum(axis=1, keepdims=True)
        return ((base * 31 + np.arange(gen)[None, :] * 7) % 1000).astype(np.int32)


def _serve_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        toks, dt, n_mine = replicas.serve(dist, 13, 4, 9, 5, 1000, _StubSession)
        q.put((rank, replicas.token_digest(toks), toks.shape, n_mine, dt))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_serve_digest_matches_single_rank():
    """The C5 serving loop (shard -> waves -> generate -> all-gather) gives the
    same token table, hence the same digest, at world 2 as at world 1."""
    toks1, _, n1 = replicas.serve(None, 13, 4, 9, 5, 1000, _StubSession)
    assert n1 == 13 and toks1.shape == (13, 5)
    want = replicas.token_digest(toks1)
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_serve_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(r[3] for r in res) == [6, 7]
    for rank, dg, shape, _, _ in res:
        assert tuple(shape) == (13, 5)
        assert dg == want
