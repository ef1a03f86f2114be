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
