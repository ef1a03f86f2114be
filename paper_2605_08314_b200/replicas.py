"""Multi-GPU plumbing for independent-request replicas.

Requests are independent and the weights are replicated, so the hot path has
no collective at all: each rank decodes its own contiguous share of the
requests. torch.distributed (NCCL on the GPU box, gloo in the CPU tests) is
used only outside the timed hot path: a start barrier, the max-over-ranks
timing reduction, and the post-run gather of generated tokens / logit
digests to rank 0.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class Rank:
    world: int
    rank: int
    local: int


def env_rank() -> Rank:
    return Rank(int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
                int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_requests: int, world: int, rank: int) -> range:
    """Contiguous request range of `rank`: sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    lo = n_requests * rank // world
    hi = n_requests * (rank + 1) // world
    return range(lo, hi)


def waves(requests: range, per_wave: int) -> list[range]:
    """Split a rank's requests into micro-batches that fit HBM."""
    if per_wave < 1:
        raise ValueError("per_wave must be >= 1")
    return [range(s, min(s + per_wave, requests.stop)) for s in range(requests.start, requests.stop, per_wave)]


def _device(pg):
    import torch

    backend = pg.get_backend()
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")


def barrier(pg) -> None:
    if pg is None:
        return
    import torch

    t = torch.zeros(1, device=_device(pg))
    pg.all_reduce(t)
    if t.is_cuda:
        torch.cuda.synchronize()


def max_over_ranks(pg, v: float) -> float:
    if pg is None:
        return v
    import torch

    t = torch.tensor([v], dtype=torch.float64, device=_device(pg))
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(pg, v: float) -> float:
    if pg is None:
        return v
    import torch

    t = torch.tensor([v], dtype=torch.float64, device=_device(pg))
    pg.all_reduce(t, op=pg.ReduceOp.SUM)
    return float(t.item())


def gather_rows(pg, rows, n_total: int):
    """All-gather per-rank [n_rank, W] int/float rows (rank order) into
    [n_total, W] on every rank; ranks may hold different row counts."""
    import torch

    if pg is None:
        return rows
    dev = _device(pg)
    world = pg.get_world_size()
    rows = rows.to(dev)
    W = rows.shape[1]
    cap = -(-n_total // world)
    buf = torch.zeros((cap, W), dtype=rows.dtype, device=dev)
    buf[: rows.shape[0]] = rows
    out = [torch.zeros_like(buf) for _ in range(world)]
    pg.all_gather(out, buf)
    parts = [out[r][: len(shard(n_total, world, r))] for r in range(world)]
    return torch.cat(parts).cpu()


def token_digest(tokens) -> str:
    """Order-sensitive digest of a [requests, gen] int32 token table (sha256 of
    the little-endian bytes, first 16 hex digits): equal digests at N = 1 and
    N > 1 mean every request produced the same tokens on every rank layout."""
    import hashlib

    import numpy as np

    a = np.ascontiguousarray(np.asarray(tokens, dtype="<i4"))
    return hashlib.sha256(a.tobytes()).hexdigest()[:16]


def request_prompt(i: int, prompt_len: int, vocab: int):
    """Prompt of request i: seeded per request (seed 2 + i)."""
    import numpy as np

    return np.random.default_rng(2 + i).integers(0, vocab, prompt_len, dtype=np.int32)


def serve(pg, n_requests: int, per_wave: int, prompt_len: int, gen: int, vocab: int, session_for, sync=None):
    """C5 serving job (BASELINE.json configs[4]): this rank's
    contiguous share of n_requests, in waves of <= per_wave, each wave one
    batched prefill + `gen` greedy steps through `session_for(B).generate`;
    then the generated tokens of every rank are all-gathered (rank order).

    Returns (tokens [n_requests, gen] on every rank, seconds = max over ranks
    of this rank's wall time, requests served by this rank). `sync()` (e.g.
    torch.cuda.synchronize) brackets the timed region. No collective runs
    inside it: the requests are independent and the weights replicated."""
    import time

    import numpy as np
    import torch

    world = pg.get_world_size() if pg is not None else 1
    rank = pg.get_rank() if pg is not None else 0
    mine = shard(n_requests, world, rank)
    toks = np.zeros((len(mine), gen), dtype=np.int32)
    prompts = {i: request_prompt(i, prompt_len, vocab) for i in mine}
    barrier(pg)
    if sync:
        sync()
    t0 = time.perf_counter()
    row = 0
    for w in waves(mine, per_wave):
        s = session_for(len(w))
        s.reset()
        out = s.generate(np.stack([prompts[i] for i in w]), gen)
        toks[row: row + len(w)] = out
        row += len(w)
    if sync:
        sync()
    dt = max_over_ranks(pg, time.perf_counter() - t0)
    allt = gather_rows(pg, torch.from_numpy(toks), n_requests)
    return np.asarray(allt), dt, len(mine)
