"""Hot-path domain types, mirroring the reference's `adaptersim.model` where the path needs them.

Time is integer microseconds (model.py:3-5, 15-16).  The byte model is the reference's
(model.py:23-26): 2 matrices x 4 projections x 32 layers x 4096 x 2 bytes = 2 MiB per unit
of rank, and an adapter occupies ceil(bytes / 512 KiB) = 4 * rank KV-token slots
(make_adapter_spec, model.py:85-93).  The enums carry the reference's string values so a
configuration built with the reference's own classes is accepted unchanged (we compare by
`.value`).
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Optional

TimePoint = int
Duration = int
US_PER_SEC = 1_000_000

DEFAULT_RANK_SET = (8, 16, 32, 64, 128)
DEFAULT_BYTES_PER_RANK_UNIT = 2 * 4 * 32 * 4096 * 2   # = 2_097_152
DEFAULT_KV_BYTES_PER_TOKEN = 524_288


class CachePolicy(Enum):
    NONE = "none"
    LRU = "lru"
    FAIRSHARE = "fairshare"
    COST_AWARE = "cost-aware"


class PrefetchMode(Enum):
    OFF = "off"
    QUEUE_DRIVEN = "queue-driven"
    HISTOGRAM = "histogram"


def enum_value(v) -> str:
    """'lru' for CachePolicy.LRU from either this module or the reference's model."""
    return getattr(v, "value", v)


@dataclass(frozen=True)
class AdapterSpec:
    adapter_id: str
    rank: int
    size_bytes: int
    size_tokens: int


def make_adapter_spec(adapter_id: str, rank: int,
                      bytes_per_rank_unit: int = DEFAULT_BYTES_PER_RANK_UNIT,
                      kv_bytes_per_token: int = DEFAULT_KV_BYTES_PER_TOKEN) -> AdapterSpec:
    """size_bytes = bytes_per_rank_unit * rank; size_tokens = max(1, ceil(size_bytes / kv))."""
    size_bytes = int(bytes_per_rank_unit) * int(rank)
    size_tokens = max(1, (size_bytes + kv_bytes_per_token - 1) // kv_bytes_per_token)
    return AdapterSpec(adapter_id, int(rank), size_bytes, size_tokens)


@dataclass
class CacheConfig:
    policy: CachePolicy = CachePolicy.COST_AWARE
    weight_frequency: float = 0.45
    weight_recency: float = 0.10
    weight_size: float = 0.45
    frequency_window_us: Duration = 60 * US_PER_SEC
    prefetch: PrefetchMode = PrefetchMode.OFF
    token_cap: Optional[int] = None


def build_catalog(num_adapters: int, rank_set=DEFAULT_RANK_SET,
                  bytes_per_rank_unit: int = DEFAULT_BYTES_PER_RANK_UNIT,
                  kv_bytes_per_token: int = DEFAULT_KV_BYTES_PER_TOKEN) -> dict[str, AdapterSpec]:
    """Ids `r{rank}-{j}`, num_adapters // len(rank_set) per rank, ranks ascending
    (workload.py:28-43)."""
    per_rank = num_adapters // len(rank_set)
    cat: dict[str, AdapterSpec] = {}
    for rank in sorted(rank_set):
        for j in range(per_rank):
            aid = f"r{rank}-{j}"
            cat[aid] = make_adapter_spec(aid, rank, bytes_per_rank_unit, kv_bytes_per_token)
    return cat


def zipf_catalog(num_adapters: int, rank_set=DEFAULT_RANK_SET, s: float = 0.7):
    """Adapter-level Zipf convention of write_mixed_trace (workload.py:220-226): adapter i
    has rank sorted(rank_set)[i % n], id r{rank}-{i // n}, popularity (i+1)^-s."""
    ranks = sorted(rank_set)
    ids, probs = [], []
    raw = [(i + 1) ** -s for i in range(num_adapters)]
    z = sum(raw)
    for i in range(num_adapters):
        rank = ranks[i % len(ranks)]
        ids.append(f"r{rank}-{i // len(ranks)}")
        probs.append(raw[i] / z)
    return ids, probs


@dataclass
class CostModelParams:
    """The reference's linear iteration-time coefficients (model.py:159-172), in microseconds;
    the adapter term is per (rank x token processed).  B200CostModel (cost_model.py) keeps the
    base-model terms and replaces the adapter term with a measured latency model."""

    prefill_base_us: float = 5_000.0
    prefill_per_token_us: float = 40.0
    decode_base_us: float = 6_000.0
    decode_per_token_us: float = 25.0
    adapter_compute_per_rank_token_us: float = 0.155
