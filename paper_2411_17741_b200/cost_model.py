"""Calibrated step-time model: the reference's linear iteration-time model with its LoRA term
replaced by the measured B200 latency of this framework's `lora_apply`.

Reference: `CostModel.step_duration` (engine.py:59-78) adds
`adapter_compute_per_rank_token_us * (Σ_decoders rank + Σ_prefills rank * input_tokens)`
(engine.py:67-77, coefficient model.py:172, "A40-calibrated" per SPEC.md:473) to the base
model's decode/prefill terms.  On B200 the apply is HBM-bound, so its latency follows the
bytes it moves, not rank x tokens: every distinct adapter of the batch is read once per
(layer, projection) and every token moves its x and y rows.  `LoraLatencyModel` therefore is

    t_us = base_us + us_per_adapter_gb * adapter_gb + us_per_token * tokens     (per path)

fitted by least squares to measured step times (`scripts/calibrate_cost.py` on the GPU box,
coefficients committed in `profiles/lora_cost_b200.json`).  `B200CostModel` keeps the
reference's method names, argument meaning and integer-µs rounding (engine.py:45-46), so the
simulator can use it in place of `CostModel`.
"""
from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field
from pathlib import Path
from typing import Iterable, Mapping, Optional, Sequence

import numpy as np

from .model import CostModelParams

ROOT = Path(__file__).resolve().parents[1]
DEFAULT_TABLE = ROOT / "profiles" / "lora_cost_b200.json"


def _round_us(x: float) -> int:
    # the reference rounds half up to integer microseconds (engine.py:45-46)
    return int(x + 0.5)


@dataclass(frozen=True)
class Geometry:
    """Model dims the adapter bytes are counted for: Llama-2-7B q/k/v/o by default (the
    reference's byte model, model.py:23-26: 2 matrices x 4 projections x 32 layers x 4096 x 2 B
    per unit of rank)."""

    n_layers: int = 32
    h_in: Sequence[int] = (4096, 4096, 4096, 4096)
    h_out: Sequence[int] = (4096, 4096, 4096, 4096)
    elem_bytes: int = 2

    def adapter_bytes(self, rank: int) -> int:
        return self.n_layers * sum(rank * (i + o) * self.elem_bytes for i, o in zip(self.h_in, self.h_out))


@dataclass
class PathCoef:
    base_us: float = 0.0
    us_per_adapter_gb: float = 0.0
    us_per_token: float = 0.0

    def __call__(self, adapter_gb: float, tokens: int) -> float:
        if tokens <= 0:
            return 0.0
        return self.base_us + self.us_per_adapter_gb * adapter_gb + self.us_per_token * tokens


@dataclass
class LoraLatencyModel:
    """Measured latency of one step's LoRA apply (all layers and projections)."""

    decode: PathCoef = field(default_factory=PathCoef)
    prefill: PathCoef = field(default_factory=PathCoef)
    geometry: Geometry = field(default_factory=Geometry)
    source: str = ""

    # -- features ----------------------------------------------------------------------
    def features(self, adapters: Iterable[str], tokens: int, rank_of: Mapping[str, int]):
        distinct = set(adapters)
        gb = sum(self.geometry.adapter_bytes(rank_of[a]) for a in distinct) / 1e9
        return gb, tokens

    def apply_us(self, decode_adapters: Sequence[str], prefills: Sequence[tuple], rank_of: Mapping[str, int]) -> float:
        """decode_adapters: one entry per decode token; prefills: (adapter_id, input_tokens)."""
        total = 0.0
        if decode_adapters:
            total += self.decode(*self.features(decode_adapters, len(decode_adapters), rank_of))
        if prefills:
            gb, _ = self.features([a for a, _ in prefills], 0, rank_of)
            total += self.prefill(gb, sum(int(n) for _, n in prefills))
        return total

    # -- persistence / calibration -----------------------------------------------------
    def to_json(self) -> dict:
        return {"decode": asdict(self.decode), "prefill": asdict(self.prefill),
                "geometry": {"n_layers": self.geometry.n_layers, "h_in": list(self.geometry.h_in),
                             "h_out": list(self.geometry.h_out), "elem_bytes": self.geometry.elem_bytes},
                "source": self.source}

    @classmethod
    def from_json(cls, d: dict) -> "LoraLatencyModel":
        g = d.get("geometry", {})
        return cls(PathCoef(**d["decode"]), PathCoef(**d["prefill"]),
                   Geometry(g.get("n_layers", 32), tuple(g.get("h_in", Geometry.h_in)),
                            tuple(g.get("h_out", Geometry.h_out)), g.get("elem_bytes", 2)),
                   d.get("source", ""))

    @classmethod
    def load(cls, path: Optional[Path] = None) -> "LoraLatencyModel":
        return cls.from_json(json.loads(Path(path or DEFAULT_TABLE).read_text()))

    @staticmethod
    def fit_path(samples: Sequence[tuple]) -> PathCoef:
        """Least squares over (adapter_gb, tokens, measured_us) samples, coefficients >= 0."""
        a = np.array([[1.0, gb, t] for gb, t, _ in samples])
        y = np.array([us for _, _, us in samples])
        coef, *_ = np.linalg.lstsq(a, y, rcond=None)
        coef = np.maximum(coef, 0.0)
        return PathCoef(float(coef[0]), float(coef[1]), float(coef[2]))


class ReferenceLoraTerm:
    """The reference's own LoRA term (engine.py:67-77): coefficient x Σ rank x tokens.  Used to
    pin `B200CostModel` to the reference's step_duration on captured batches."""

    def __init__(self, per_rank_token_us: float):
        self.c = per_rank_token_us

    def apply_us(self, decode_adapters, prefills, rank_of) -> float:
        units = sum(rank_of[a] for a in decode_adapters) + sum(rank_of[a] * int(n) for a, n in prefills)
        return self.c * units


class B200CostModel:
    """Drop-in for the reference `CostModel` (engine.py:53-97): same methods, same base-model
    terms, the LoRA term from a measured B200 latency model."""

    def __init__(self, params: CostModelParams, lora=None):
        self.p = params
        self.lora = lora if lora is not None else LoraLatencyModel.load()

    def _base(self, prefills, decoders) -> float:
        p = self.p
        total = p.decode_base_us
        active = sum(r.spec.input_tokens + r.tokens_generated for r in decoders)
        total += p.decode_per_token_us * active
        if prefills:
            total += p.prefill_base_us + sum(p.prefill_per_token_us * r.spec.input_tokens for r in prefills)
        return total

    def step_duration(self, prefills, decoders, rank_of) -> int:
        lora = self.lora.apply_us([r.spec.adapter_id for r in decoders],
                                  [(r.spec.adapter_id, r.spec.input_tokens) for r in prefills], rank_of)
        return _round_us(self._base(prefills, decoders) + lora)

    def prefill_step_us(self, input_tokens: int, rank: int, adapter_id: str = "a") -> int:
        p = self.p
        lora = self.lora.apply_us([], [(adapter_id, input_tokens)], {adapter_id: rank})
        return _round_us(p.decode_base_us + p.prefill_base_us + p.prefill_per_token_us * input_tokens + lora)

    def decode_steps_us(self, input_tokens: int, output_tokens: int, rank: int, adapter_id: str = "a") -> int:
        """Sum of the solo decode iterations for tokens 2..output_tokens (engine.py:89-97)."""
        if output_tokens <= 1:
            return 0
        p = self.p
        lora = self.lora.apply_us([adapter_id], [], {adapter_id: rank})
        g = np.arange(1, output_tokens)
        steps = np.floor(p.decode_base_us + lora + p.decode_per_token_us * (input_tokens + g) + 0.5)
        return int(steps.sum())
