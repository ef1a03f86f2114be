"""Greedy-decode fidelity audit (SPEC.md:503-511 audit_fidelity; the paper's
Table 4): N seeded prompts (lengths uniform in [16, 128]), each
decoded greedily for `max_new` tokens by candidate systems and compared with
gold token sequences.

The product side only generates candidates (through the C ABI) and scores
them; the gold sequences are an input. The f64 no-cache gold of the SPEC is
produced by the CPU oracle in tests/ and tools/ (test infrastructure) -- this
module never imports it.
"""
from __future__ import annotations

from dataclasses import asdict, dataclass

import numpy as np

_MASK = (1 << 64) - 1


class Rng64:
    """SplitMix64 of tensor.hpp:35-62 (next_u64 / next_unit / next_below)."""

    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def next_unit(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def next_below(self, n: int) -> int:
        return int(self.next_unit() * float(n))


def audit_prompts(n_prompts: int, vocab: int, seed: int = 2, min_len: int = 16, max_len: int = 128) -> list:
    """Seeded prompts: length uniform in [min_len, max_len], tokens uniform in [0, vocab)."""
    rng = Rng64(seed)
    out = []
    for _ in range(n_prompts):
        T = min_len + rng.next_below(max_len - min_len + 1)
        out.append(np.array([rng.next_below(vocab) for _ in range(T)], dtype=np.int32))
    return out


@dataclass
class AuditReport:
    """SPEC.md:461-464 AuditReport (k/N counts, mean token match in [0, 1])."""

    n_prompts: int
    max_new: int
    exact_match: int
    first_token_match: int
    mean_token_match: float
    pairwise_exact: int | None = None

    def as_dict(self) -> dict:
        return asdict(self)


def score(gold: list, cand: list, other: list | None = None) -> AuditReport:
    """Compare candidate greedy sequences with gold ones (and, optionally, a
    second candidate for the pairwise-exact count)."""
    if len(gold) != len(cand) or (other is not None and len(other) != len(cand)):
        raise ValueError("gold / candidate prompt counts differ")
    n = len(gold)
    max_new = len(gold[0]) if n else 0
    exact = sum(int(np.array_equal(g, c)) for g, c in zip(gold, cand))
    first = sum(int(g[0] == c[0]) for g, c in zip(gold, cand))
    mean = float(np.mean([np.mean(np.asarray(g) == np.asarray(c)) for g, c in zip(gold, cand)])) if n else 1.0
    pair = None if other is None else sum(int(np.array_equal(a, b)) for a, b in zip(cand, other))
    return AuditReport(n, max_new, exact, first, mean, pair)


def generate_candidates(model, prompts: list, max_new: int, plan: str = "eager", capacity: int = 0) -> list:
    """Greedy decode of every prompt (batch 1, one session per prompt length)
    on the GPU through the C ABI."""
    import paper_2605_08314_b200 as F

    cap = capacity or (max(len(p) for p in prompts) + max_new + 8)
    out = []
    s = F.Session(model, batch=1, capacity=cap, plan=plan)
    for p in prompts:
        s.reset()
        out.append(s.generate(p[None], max_new)[0].copy())
    return out
