"""Reference-facing operators: `build_segments` and `lora_apply`.

`lora_apply(x, y, slot_ids, seg_offsets, ranks, ...)` is the drop-in operator for the
reference seam `CostModel.step_duration` (engine.py:59-78), whose LoRA term
`adapter_compute_per_rank_token_us * adapter_units` (engine.py:67-77) models exactly the
work this operator performs on the GPU.  All arithmetic runs in the sm_100a kernels of
`libchameleon_lora.so`; there is no CPU fallback (a missing extension raises ChamError).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _lib
from ._lib import call
from .pool import AdapterPool, _stream_ptr


@dataclass
class SegmentTable:
    """Device-resident grouped batch: perm [T], seg_off [S+1], seg_slot [S], seg_rank [S],
    n_seg [1] (device), n_tokens (host).  Capacity rows beyond n_seg are unused."""

    perm: torch.Tensor
    seg_off: torch.Tensor
    seg_slot: torch.Tensor
    seg_rank: torch.Tensor
    n_seg: torch.Tensor
    n_tokens: int
    n_seg_host: Optional[int] = None
    plan: Optional[torch.Tensor] = None  # device launch plan (build_plan), valid for one step

    def to_host(self):
        """(perm, seg_off, seg_slot, seg_rank) trimmed to the real segment count, numpy."""
        S = int(self.n_seg.item()) if self.n_seg_host is None else self.n_seg_host
        off = self.seg_off[: S + 1].cpu().numpy()
        n = int(off[-1]) if S >= 0 else 0
        return (self.perm[:n].cpu().numpy(), off, self.seg_slot[:S].cpu().numpy(),
                self.seg_rank[:S].cpu().numpy())


def _i32(t, device) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(t, dtype=torch.int32)
    return t.to(device=device, dtype=torch.int32).contiguous()


def build_segments(req_slot, req_rank, req_ntok, *, device=None, stream=None,
                   out: Optional[SegmentTable] = None) -> SegmentTable:
    """Device-side (K4) stable group-by-slot of a batch of requests.

    Requests are in batch order (the reference's `(ready_prefills, decoding)`,
    engine.py:443-451): request i owns the next `req_ntok[i]` token rows.  Returns the
    segment table in canonical order (ascending slot, ties in batch order).
    """
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    rs = _i32(req_slot, device)
    rr = _i32(req_rank, device)
    rn = _i32(req_ntok, device)
    n_req = rs.numel()
    if n_req > _lib.limits().max_requests:
        raise ValueError(f"batch of {n_req} requests exceeds max_requests={_lib.limits().max_requests}")
    if isinstance(req_ntok, torch.Tensor) and req_ntok.device.type != "cpu":
        n_tok = None
    else:
        n_tok = int(sum(int(v) for v in (req_ntok.tolist() if hasattr(req_ntok, "tolist") else req_ntok)))
    if out is None:
        cap_tok = n_tok if n_tok is not None else int(rn.sum().item())
        out = SegmentTable(
            perm=torch.empty(max(cap_tok, 1), dtype=torch.int32, device=device),
            seg_off=torch.empty(n_req + 1, dtype=torch.int32, device=device),
            seg_slot=torch.empty(max(n_req, 1), dtype=torch.int32, device=device),
            seg_rank=torch.empty(max(n_req, 1), dtype=torch.int32, device=device),
            n_seg=torch.empty(1, dtype=torch.int32, device=device),
            n_tokens=cap_tok,
        )
    call("cham_build_segments", rs.data_ptr(), rr.data_ptr(), rn.data_ptr(), n_req, out.perm.data_ptr(),
         out.seg_off.data_ptr(), out.seg_slot.data_ptr(), out.seg_rank.data_ptr(), out.n_seg.data_ptr(),
         _stream_ptr(stream))
    return out


def plan_bytes(pool: AdapterPool) -> int:
    return int(_lib.lib().cham_plan_bytes(pool.handle))


def build_plan(table: SegmentTable, *, pool: AdapterPool, stream=None) -> torch.Tensor:
    """Device launch plan for `table` against the pool's slot table (one CTA).  Every
    lora_apply of the step reuses it, so the kernels skip their own plan construction."""
    if table.plan is None:
        table.plan = torch.empty(plan_bytes(pool), dtype=torch.uint8, device=pool.device)
    call("cham_build_plan", pool.handle, table.perm.data_ptr(), table.seg_off.data_ptr(), table.seg_slot.data_ptr(),
         table.seg_rank.data_ptr(), -1 if table.n_seg_host is None else table.n_seg_host, table.n_seg.data_ptr(),
         table.plan.data_ptr(), _stream_ptr(stream))
    return table.plan


def _check_act(t: torch.Tensor, pool: AdapterPool, cols: int, name: str) -> None:
    if t.device != pool.device:
        raise ValueError(f"{name} must live on {pool.device}")
    if t.dtype != pool.dtype:
        raise ValueError(f"{name} dtype {t.dtype} != pool dtype {pool.dtype}")
    if t.dim() != 2 or t.shape[1] != cols or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous [T, {cols}] tensor")


def _tables(slot_ids, seg_offsets, ranks, perm, device):
    return (_i32(slot_ids, device), _i32(seg_offsets, device), _i32(ranks, device),
            None if perm is None else _i32(perm, device))


def lora_apply(x: torch.Tensor, y: torch.Tensor, slot_ids, seg_offsets, ranks, *, pool: AdapterPool,
               layer: int, proj: int, perm=None, n_seg: Optional[int] = None, n_seg_dev=None,
               plan: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """y[t] += (x[t] . A_slot) . B_slot for every token of every segment (in place).

    x: [T, h_in[proj]], y: [T, h_out[proj]] in the pool dtype on the pool device.
    slot_ids [S], seg_offsets [S+1], ranks [S]: the segment table (segment s covers grouped
    positions seg_offsets[s]..seg_offsets[s+1]; perm maps grouped position -> token row,
    None = identity).  With `n_seg_dev` (device int32 [1]) the segment count is read on the
    device, so the call is CUDA-graph capturable without a host sync.
    """
    _check_act(x, pool, pool.h_in[proj], "x")
    _check_act(y, pool, pool.h_out[proj], "y")
    if x.shape[0] != y.shape[0]:
        raise ValueError("x and y must have the same number of token rows")
    ss, so, sr, pm = _tables(slot_ids, seg_offsets, ranks, perm, pool.device)
    if n_seg is None and n_seg_dev is None:
        n_seg = ss.numel()
    call("cham_lora_apply", pool.handle, int(layer), int(proj), x.data_ptr(), y.data_ptr(), int(x.shape[0]),
         _lib.ptr(pm), so.data_ptr(), ss.data_ptr(), sr.data_ptr(), -1 if n_seg is None else int(n_seg),
         _lib.ptr(n_seg_dev), _lib.ptr(plan), _stream_ptr(stream))
    return y


def lora_apply_table(x, y, table: SegmentTable, *, pool: AdapterPool, layer: int, proj: int, stream=None):
    """lora_apply driven by a device SegmentTable (count read on the device)."""
    _check_act(x, pool, pool.h_in[proj], "x")
    _check_act(y, pool, pool.h_out[proj], "y")
    call("cham_lora_apply", pool.handle, int(layer), int(proj), x.data_ptr(), y.data_ptr(), int(x.shape[0]),
         table.perm.data_ptr(), table.seg_off.data_ptr(), table.seg_slot.data_ptr(), table.seg_rank.data_ptr(),
         -1 if table.n_seg_host is None else table.n_seg_host, table.n_seg.data_ptr(), _lib.ptr(table.plan),
         _stream_ptr(stream))
    return y


def lora_apply_multi(xs: Sequence[torch.Tensor], ys: Sequence[torch.Tensor], table: SegmentTable, *,
                     pool: AdapterPool, layer: int, projs: Sequence[int], stream=None):
    """Several projections of one layer sharing the token batch (q/k/v) in ONE launch."""
    if not (len(xs) == len(ys) == len(projs)):
        raise ValueError("xs, ys and projs must have equal length")
    for x, y, p in zip(xs, ys, projs):
        _check_act(x, pool, pool.h_in[p], "x")
        _check_act(y, pool, pool.h_out[p], "y")
    n = len(projs)
    xa = (ctypes.c_void_p * n)(*[x.data_ptr() for x in xs])
    ya = (ctypes.c_void_p * n)(*[y.data_ptr() for y in ys])
    call("cham_lora_apply_multi", pool.handle, int(layer), n, _lib.int_array(projs), xa, ya, int(xs[0].shape[0]),
         table.perm.data_ptr(), table.seg_off.data_ptr(), table.seg_slot.data_ptr(), table.seg_rank.data_ptr(),
         -1 if table.n_seg_host is None else table.n_seg_host, table.n_seg.data_ptr(), _lib.ptr(table.plan),
         _stream_ptr(stream))


def lora_apply_multi_arrays(xs: Sequence[torch.Tensor], ys: Sequence[torch.Tensor], slot_ids, seg_offsets, ranks, *,
                            pool: AdapterPool, layer: int, projs: Sequence[int], perm=None,
                            n_seg: Optional[int] = None, plan=None, stream=None):
    """lora_apply_multi over explicit segment arrays (projections sharing h_in and h_out)."""
    if not (len(xs) == len(ys) == len(projs)):
        raise ValueError("xs, ys and projs must have equal length")
    for x, y, p in zip(xs, ys, projs):
        _check_act(x, pool, pool.h_in[p], "x")
        _check_act(y, pool, pool.h_out[p], "y")
    ss, so, sr, pm = _tables(slot_ids, seg_offsets, ranks, perm, pool.device)
    n = len(projs)
    xa = (ctypes.c_void_p * n)(*[x.data_ptr() for x in xs])
    ya = (ctypes.c_void_p * n)(*[y.data_ptr() for y in ys])
    call("cham_lora_apply_multi", pool.handle, int(layer), n, _lib.int_array(projs), xa, ya, int(xs[0].shape[0]),
         _lib.ptr(pm), so.data_ptr(), ss.data_ptr(), sr.data_ptr(), ss.numel() if n_seg is None else int(n_seg),
         None, _lib.ptr(plan), _stream_ptr(stream))


def _check_v(v: torch.Tensor) -> None:
    """v: fp32 [positions, cols] with unit column stride; the row stride (a multiple of 4
    floats, 16-byte aligned base) is passed as v_stride, so a column slice of a wider
    buffer (the fused q/k/v operand of one all-reduce) is accepted.  The kernels write and
    read ranks up to the segment's padded rank: cols must cover it."""
    if v.dtype != torch.float32 or v.dim() != 2 or v.stride(1) != 1:
        raise ValueError("v must be an fp32 [positions, cols] tensor with unit column stride")
    if v.stride(0) % 4 or v.data_ptr() % 16:
        raise ValueError("v rows must be 16-byte aligned (row stride a multiple of 4 floats)")


def lora_shrink(x: torch.Tensor, v: torch.Tensor, slot_ids, seg_offsets, ranks, *, pool: AdapterPool,
                layer: int, proj: int, perm=None, n_seg: Optional[int] = None, plan=None,
                stream=None) -> torch.Tensor:
    """v[k, :r] = x[perm[k]] . A_slot (fp32 [n_positions, v_stride]); the TP all-reduce operand."""
    _check_act(x, pool, pool.h_in[proj], "x")
    _check_v(v)
    ss, so, sr, pm = _tables(slot_ids, seg_offsets, ranks, perm, pool.device)
    call("cham_lora_shrink", pool.handle, int(layer), int(proj), x.data_ptr(), v.data_ptr(), int(v.stride(0)),
         int(x.shape[0]), _lib.ptr(pm), so.data_ptr(), ss.data_ptr(), sr.data_ptr(),
         ss.numel() if n_seg is None else int(n_seg), None, _lib.ptr(plan), _stream_ptr(stream))
    return v


def lora_expand(v: torch.Tensor, y: torch.Tensor, slot_ids, seg_offsets, ranks, *, pool: AdapterPool,
                layer: int, proj: int, perm=None, n_seg: Optional[int] = None, plan=None,
                stream=None) -> torch.Tensor:
    """y[perm[k]] += v[k, :r] . B_slot (in place)."""
    _check_act(y, pool, pool.h_out[proj], "y")
    _check_v(v)
    ss, so, sr, pm = _tables(slot_ids, seg_offsets, ranks, perm, pool.device)
    call("cham_lora_expand", pool.handle, int(layer), int(proj), v.data_ptr(), int(v.stride(0)), y.data_ptr(),
         int(y.shape[0]), _lib.ptr(pm), so.data_ptr(), ss.data_ptr(), sr.data_ptr(),
         ss.numel() if n_seg is None else int(n_seg), None, _lib.ptr(plan), _stream_ptr(stream))
    return y


def _multi_v_check(v: torch.Tensor, n: int) -> int:
    """v: the fused fp32 [positions, n * v_cols] buffer (column slice views accepted)."""
    _check_v(v)
    if v.shape[1] % n or (v.shape[1] // n) % 4:
        raise ValueError("v columns must split into len(projs) slices of a multiple of 4 columns")
    return v.shape[1] // n


def lora_shrink_multi(xs: Sequence[torch.Tensor], v: torch.Tensor, slot_ids, seg_offsets, ranks, *,
                      pool: AdapterPool, layer: int, projs: Sequence[int], perm=None, n_seg: Optional[int] = None,
                      plan=None, stream=None) -> torch.Tensor:
    """v[k, j*c:(j+1)*c][:r] = x_j[perm[k]] . A_slot(projs[j]) for every j in ONE launch, c =
    v.shape[1] / len(projs) (the TP all-reduce operand of a projection group sharing h_in)."""
    n = len(projs)
    if len(xs) != n:
        raise ValueError("xs and projs must have equal length")
    for x, p in zip(xs, projs):
        _check_act(x, pool, pool.h_in[p], "x")
    cols = _multi_v_check(v, n)
    ss, so, sr, pm = _tables(slot_ids, seg_offsets, ranks, perm, pool.device)
    xa = (ctypes.c_void_p * n)(*[x.data_ptr() for x in xs])
    call("cham_lora_shrink_multi", pool.handle, int(layer), n, _lib.int_array(projs), xa, v.data_ptr(),
         int(v.stride(0)), cols, int(xs[0].shape[0]), _lib.ptr(pm), so.data_ptr(), ss.data_ptr(), sr.data_ptr(),
         ss.numel() if n_seg is None else int(n_seg), None, _lib.ptr(plan), _stream_ptr(stream))
    return v


def lora_expand_multi(v: torch.Tensor, ys: Sequence[torch.Tensor], slot_ids, seg_offsets, ranks, *,
                      pool: AdapterPool, layer: int, projs: Sequence[int], perm=None, n_seg: Optional[int] = None,
                      plan=None, stream=None):
    """y_j[perm[k]] += v[k, j*c:(j+1)*c] . B_slot(projs[j]) for every j in ONE launch (shared h_out)."""
    n = len(projs)
    if len(ys) != n:
        raise ValueError("ys and projs must have equal length")
    for y, p in zip(ys, projs):
        _check_act(y, pool, pool.h_out[p], "y")
    cols = _multi_v_check(v, n)
    ss, so, sr, pm = _tables(slot_ids, seg_offsets, ranks, perm, pool.device)
    ya = (ctypes.c_void_p * n)(*[y.data_ptr() for y in ys])
    call("cham_lora_expand_multi", pool.handle, int(layer), n, _lib.int_array(projs), v.data_ptr(), int(v.stride(0)),
         cols, ya, int(ys[0].shape[0]), _lib.ptr(pm), so.data_ptr(), ss.data_ptr(), sr.data_ptr(),
         ss.numel() if n_seg is None else int(n_seg), None, _lib.ptr(plan), _stream_ptr(stream))
