"""Numpy restatement of the segment-table builder (test infrastructure only).

The reference has no segment concept; its per-step batch is `(ready_prefills, decoding)`
(engine.py:443-451) and CostModel.step_duration walks it request by request, attributing
`input_tokens` tokens to a prefill and 1 token to a decoder (engine.py:64-76).  The
canonical table: requests in batch order own consecutive token rows; a stable
sort of requests by slot (ties keep batch order) gives `perm`; run-length encoding of the
sorted slots gives seg_off / seg_slot / seg_rank.  Requests with slot < 0 have no adapter.
"""
from __future__ import annotations

import numpy as np


def build_segments_ref(req_slot, req_rank, req_ntok):
    req_slot = np.asarray(req_slot, dtype=np.int64)
    req_rank = np.asarray(req_rank, dtype=np.int64)
    req_ntok = np.maximum(np.asarray(req_ntok, dtype=np.int64), 0)
    n = len(req_slot)
    tok_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(req_ntok, out=tok_off[1:])
    valid = req_slot >= 0
    idx = np.nonzero(valid)[0]
    order = idx[np.argsort(req_slot[idx], kind="stable")]
    perm = np.concatenate([np.arange(tok_off[i], tok_off[i] + req_ntok[i]) for i in order]) \
        if len(order) else np.zeros(0, dtype=np.int64)
    seg_off, seg_slot, seg_rank = [], [], []
    pos = 0
    prev = None
    for i in order:
        s = int(req_slot[i])
        if s != prev:
            seg_off.append(pos)
            seg_slot.append(s)
            seg_rank.append(int(req_rank[i]))
            prev = s
        pos += int(req_ntok[i])
    seg_off.append(pos)
    return (perm.astype(np.int32), np.asarray(seg_off, dtype=np.int32),
            np.asarray(seg_slot, dtype=np.int32), np.asarray(seg_rank, dtype=np.int32))


def adapter_units(req_rank, req_ntok):
    """sum_i rank_i * tokens_i — the reference's `adapter_units` (engine.py:64-76)."""
    return int(np.sum(np.asarray(req_rank, dtype=np.int64) * np.asarray(req_ntok, dtype=np.int64)))
