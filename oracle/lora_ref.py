"""Numpy restatement of the batched heterogeneous-rank LoRA apply (test infrastructure only).

Definition (BASELINE.json north_star): for every token t of every segment s,
    y[t] += (x[t] . A_{slot(s)}) . B_{slot(s)}
with A_i of shape [h_in, r_i] and B_i of shape [r_i, h_out] (the byte model of
model.py:23-26: two matrices per projection).  Token -> rank attribution follows the
reference cost model: a decoder contributes 1 token, a prefill `input_tokens` tokens
(engine.py:64-76).

The reference never computes this product (SPEC.md:12 puts GPU kernels out of scope;
PAPER.md:139-141 delegates them to third-party S-LoRA, not vendored).  This restatement is
pinned instead to third-party golden vectors: vLLM 0.22.0's torch Punica SGMV shrink/expand
(the published algorithm S-LoRA implements), tests/golden/punica_sgmv.npz made by
oracle/punica_golden.py and checked in tests/test_punica_golden.py.
"""
from __future__ import annotations

import numpy as np


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even); returns float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    nan = np.isnan(a)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    out = u.astype(np.uint32).view(np.float32).copy()
    out[nan] = np.nan
    return out


def bf16_bits(a: np.ndarray) -> np.ndarray:
    """float32 -> uint16 bit pattern of the bf16 rounding."""
    return (bf16_round(a).view(np.uint32) >> 16).astype(np.uint16)


def bf16_from_bits(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def lora_apply_ref(x, y, perm, seg_off, seg_slot, seg_rank, adapters, *, acc=np.float64):
    """Return y + LoRA(x) as `acc` dtype (y itself is not modified).

    x: [T, h_in]; y: [T, h_out]; perm: [P] grouped position -> token row (None = identity);
    seg_off: [S+1]; seg_slot, seg_rank: [S]; adapters: slot -> (A [h_in, r], B [r, h_out]).
    Only the first seg_rank[s] columns of A / rows of B take part (pool rows beyond the rank
    are zero padding).  Segments with slot < 0 carry no adapter.
    """
    x = np.asarray(x, dtype=acc)
    out = np.array(y, dtype=acc, copy=True)
    n_seg = len(seg_slot)
    for s in range(n_seg):
        slot = int(seg_slot[s])
        if slot < 0:
            continue
        lo, hi = int(seg_off[s]), int(seg_off[s + 1])
        if hi <= lo:
            continue
        rows = np.arange(lo, hi) if perm is None else np.asarray(perm[lo:hi], dtype=np.int64)
        a, b = adapters[slot]
        r = int(seg_rank[s])
        v = x[rows] @ np.asarray(a, dtype=acc)[:, :r]
        out[rows] += v @ np.asarray(b, dtype=acc)[:r, :]
    return out


def lora_shrink_ref(x, perm, seg_off, seg_slot, seg_rank, adapters, r_stride, *, acc=np.float64):
    """v[k, 0:r] = x[perm[k]] . A_slot for every grouped position k (rows beyond r are 0)."""
    x = np.asarray(x, dtype=acc)
    n_pos = int(seg_off[len(seg_slot)]) if len(seg_slot) else 0
    v = np.zeros((n_pos, r_stride), dtype=acc)
    for s in range(len(seg_slot)):
        slot = int(seg_slot[s])
        lo, hi = int(seg_off[s]), int(seg_off[s + 1])
        if slot < 0 or hi <= lo:
            continue
        rows = np.arange(lo, hi) if perm is None else np.asarray(perm[lo:hi], dtype=np.int64)
        a, _ = adapters[slot]
        r = int(seg_rank[s])
        v[lo:hi, :r] = x[rows] @ np.asarray(a, dtype=acc)[:, :r]
    return v


def lora_expand_ref(v, y, perm, seg_off, seg_slot, seg_rank, adapters, *, acc=np.float64):
    out = np.array(y, dtype=acc, copy=True)
    v = np.asarray(v, dtype=acc)
    for s in range(len(seg_slot)):
        slot = int(seg_slot[s])
        lo, hi = int(seg_off[s]), int(seg_off[s + 1])
        if slot < 0 or hi <= lo:
            continue
        rows = np.arange(lo, hi) if perm is None else np.asarray(perm[lo:hi], dtype=np.int64)
        _, b = adapters[slot]
        r = int(seg_rank[s])
        out[rows] += v[lo:hi, :r] @ np.asarray(b, dtype=acc)[:r, :]
    return out


def make_adapters(rng, slot_ranks, h_in, h_out, dtype=np.float32, bf16=False):
    """Synthetic random-init adapters: A ~ N(0, 1/h_in), B ~ N(0, 1/r)."""
    out = {}
    for slot, r in slot_ranks.items():
        a = (rng.standard_normal((h_in, r)) / np.sqrt(h_in)).astype(np.float32)
        b = (rng.standard_normal((r, h_out)) / np.sqrt(r)).astype(np.float32)
        if bf16:
            a, b = bf16_round(a), bf16_round(b)
        out[slot] = (a.astype(dtype), b.astype(dtype))
    return out


def algorithmic_bytes(seg_off, seg_slot, seg_rank, n_tokens, h_in, h_out, w_bytes, x_bytes, y_bytes):
    """distinct adapters once per (layer, proj) + T*(h_in*s_x + 2*h_out*s_y)."""
    seen = {}
    for s in range(len(seg_slot)):
        if seg_slot[s] >= 0 and seg_off[s + 1] > seg_off[s]:
            seen[int(seg_slot[s])] = int(seg_rank[s])
    adapter = sum(r * (h_in + h_out) * w_bytes for r in seen.values())
    act = n_tokens * (h_in * x_bytes + 2 * h_out * y_bytes)
    return adapter, act
