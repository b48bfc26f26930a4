"""Synthetic batch generators for the LoRA-apply benchmarks (the reference's L1 input side).

Restates the reference generators that define the BASELINE configs (SURVEY §8a rows
a22-a23), so the GPU box can rebuild the exact workloads without the reference package:
  * rank_probabilities / assign_adapter (workload.py:46-64): rank index i drawn with
    P(i) ∝ (i+1)^-s, then an adapter of that rank uniformly;
  * adapter-level Zipf ids (write_mixed_trace, workload.py:220-226) — see model.zipf_catalog.
tests/golden/workload_draws.json (generated from the reference) pins both bit-exactly.
"""
from __future__ import annotations

import numpy as np

from .model import DEFAULT_RANK_SET, build_catalog, zipf_catalog


def rank_probabilities(rank_set=DEFAULT_RANK_SET, s: float = 1.0) -> list[float]:
    weights = [(i + 1) ** -s for i in range(len(rank_set))]
    total = sum(weights)
    return [w / total for w in weights]


def assign_adapter(rng: np.random.Generator, num_adapters: int = 100, rank_set=DEFAULT_RANK_SET,
                   s: float = 1.0) -> str:
    ranks = sorted(rank_set)
    rank = ranks[rng.choice(len(ranks), p=rank_probabilities(rank_set, s))]
    per_rank = num_adapters // len(ranks)
    j = int(rng.integers(per_rank))
    return f"r{rank}-{j}"


def decode_batch(seed: int, n_tokens: int = 256, num_adapters: int = 100, rank_set=DEFAULT_RANK_SET):
    """C2: one decode token per request, adapters by assign_adapter(default_rng(seed))."""
    rng = np.random.default_rng(seed)
    return [assign_adapter(rng, num_adapters, rank_set) for _ in range(n_tokens)]


def zipf_batch(seed: int, n_tokens: int = 256, num_adapters: int = 1000, rank_set=DEFAULT_RANK_SET,
               s: float = 0.7):
    """C4: adapter-level Zipf draws (write_mixed_trace convention)."""
    ids, probs = zipf_catalog(num_adapters, rank_set, s)
    rng = np.random.default_rng(seed)
    return [ids[int(rng.choice(num_adapters, p=probs))] for _ in range(n_tokens)]


def prefill_batch(seed: int, n_segments: int = 64, tokens_per_segment: int = 64, num_adapters: int = 100,
                  rank_set=DEFAULT_RANK_SET):
    """C3: n_segments prefill requests of tokens_per_segment tokens, one distinct adapter each
    (BASELINE.json C3: 64 segments / 64 adapters).  Ranks are drawn directly with the s=1
    power law from default_rng(seed) (seed 0: sum of ranks 1,864); the j-th
    adapter of rank r is `r{r}-{j}`."""
    ranks = sorted(rank_set)
    rng = np.random.default_rng(seed)
    draws = rng.choice(len(ranks), n_segments, p=rank_probabilities(rank_set))
    count: dict[int, int] = {}
    ids = []
    for i in draws:
        r = ranks[int(i)]
        ids.append(f"r{r}-{count.get(r, 0)}")
        count[r] = count.get(r, 0) + 1
    return ids, [tokens_per_segment] * n_segments


def rank_of_id(adapter_id: str) -> int:
    return int(adapter_id[1:].split("-")[0])


__all__ = ["rank_probabilities", "assign_adapter", "decode_batch", "zipf_batch", "prefill_batch",
           "build_catalog", "rank_of_id"]
