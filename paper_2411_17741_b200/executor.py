"""Step executor: the device-side replacement of the reference's LoRA cost seam.

In the reference, one engine step is `(prefills, decoders) = (ready_prefills, decoding)`
(engine.py:443-451) and its LoRA work is only *modelled* by CostModel.step_duration
(engine.py:59-78).  `LoraStepExecutor` executes that work: it turns the batch descriptor
into per-request (slot, rank, tokens) arrays, uploads them (pinned, async), builds the
segment table on the device (K4) and runs `lora_apply` for every (layer, projection
group).  The whole device part is stream-ordered and CUDA-graph capturable (the segment
count never leaves the device), so a step replays as one graph.
"""
from __future__ import annotations

import os
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import _lib
from .ops import SegmentTable, build_plan, build_segments, lora_apply_multi, lora_apply_table
from .pool import AdapterPool


DEFAULT_L2_PREFETCH_MB = 0


def batch_arrays(batch, slot_of: Callable[[str], int], rank_of: Callable[[str], int]):
    """Per-request (slot, rank, tokens) arrays in batch order.

    `batch` is either the engine's step tuple `(prefills, decoders)` — prefills contribute
    `spec.input_tokens` tokens, decoders 1 token (engine.py:64-76) — or a list of admitted
    requests (`BatchResult.admitted`, scheduler.py:246-255), which enter as prefills.
    Objects are duck-typed: anything with `.spec.adapter_id` and `.spec.input_tokens`.
    """
    if isinstance(batch, tuple) and len(batch) == 2:
        prefills, decoders = batch
    else:
        prefills, decoders = list(batch), []
    slots, ranks, ntok = [], [], []
    for r in prefills:
        aid = r.spec.adapter_id
        slots.append(slot_of(aid))
        ranks.append(rank_of(aid))
        ntok.append(int(r.spec.input_tokens))
    for r in decoders:
        aid = r.spec.adapter_id
        slots.append(slot_of(aid))
        ranks.append(rank_of(aid))
        ntok.append(1)
    return (np.asarray(slots, dtype=np.int32), np.asarray(ranks, dtype=np.int32),
            np.asarray(ntok, dtype=np.int32))


def segment_token_bounds(req_slot, req_rank, req_ntok, max_rank: int = 128) -> tuple[int, int]:
    """(min, max) tokens over the step's segments (one segment per distinct slot >= 0), the
    routing hints of cham_pool_set_prefill_route.  A segment whose rank exceeds the tcgen05
    path's limit forces min = 0 (it needs the decode kernel).  Vectorised, no per-request loop."""
    slot = np.asarray(req_slot, dtype=np.int64)
    ntok = np.asarray(req_ntok, dtype=np.int64)
    rank = np.asarray(req_rank, dtype=np.int64)
    m = slot >= 0
    if not m.any():
        return 0, 0
    tok = np.bincount(slot[m], weights=ntok[m]).astype(np.int64)
    present = np.bincount(slot[m]) > 0
    seg = tok[present]
    lo, hi = int(seg.min()), int(seg.max())
    if (rank[m] > max_rank).any():
        lo = 0
    return lo, hi


def adapter_units(batch, rank_of: Callable[[str], int]) -> int:
    """The reference's `adapter_units` of a step (engine.py:64-76), as an integer."""
    _, ranks, ntok = batch_arrays(batch, lambda a: 0, rank_of)
    return int(np.sum(ranks.astype(np.int64) * ntok))


class LoraStepExecutor:
    """Runs one step's LoRA work on one replica.

    proj_groups: projections that share their input activation and run in one launch
    (e.g. [[0, 1, 2], [3]] for q/k/v + o); default: every projection on its own.
    """

    def __init__(self, pool: AdapterPool, max_requests: int = 4096, max_tokens: Optional[int] = None,
                 proj_groups: Optional[Sequence[Sequence[int]]] = None, stream=None, prefill_min_tokens: int = 64,
                 route_hints: bool = True, graph_requests: Optional[int] = None,
                 l2_prefetch_bytes: Optional[int] = None):
        """graph_requests: pad every upload to this many requests (slot -1, 0 tokens — K4 drops
        them, so the segment table is unchanged) so that one captured step graph, whose K4
        launch bakes in the request count, replays any batch of up to that many requests."""
        self.pool = pool
        # cross-apply prefetch: each apply pulls the first l2_prefetch_bytes of the NEXT
        # (layer, group) apply's A blocks into L2 once it runs out of units (its tail and the
        # launch boundary leave HBM idle).  Env CHAM_L2_PREFETCH_MB overrides the default.
        if l2_prefetch_bytes is None:
            l2_prefetch_bytes = int(float(os.environ.get("CHAM_L2_PREFETCH_MB", DEFAULT_L2_PREFETCH_MB)) * (1 << 20))
        self.l2_prefetch_bytes = int(l2_prefetch_bytes)
        pool.set_l2_prefetch(self.l2_prefetch_bytes)
        # tcgen05 routing: segments >= prefill_min_tokens (bf16 pools; 0 disables).  With
        # route_hints the host passes each step's segment-length bounds, so only the kernel
        # family with work is launched (set before the step's plan is built / captured).
        self.prefill_min_tokens = int(prefill_min_tokens) if pool.dtype == torch.bfloat16 else 0
        self.route_hints = route_hints
        self.prefill_launched = False
        self.decode_launched = True
        pool.set_prefill_route(self.prefill_min_tokens)
        dev = pool.device
        self.max_requests = min(int(max_requests), _lib.limits().max_requests)
        self.max_tokens = int(max_tokens or pool.max_tokens)
        self.proj_groups = [list(g) for g in (proj_groups or [[p] for p in range(pool.n_proj)])]
        self.stream = stream
        if graph_requests is not None and not 0 < int(graph_requests) <= self.max_requests:
            raise ValueError(f"graph_requests must be in [1, {self.max_requests}]")
        self.graph_requests = None if graph_requests is None else int(graph_requests)
        self.req_dev = torch.zeros(3, self.max_requests, dtype=torch.int32, device=dev)
        # two pinned staging buffers, each reused only after its previous H2D copy completed
        self._req_host = [torch.zeros(3, self.max_requests, dtype=torch.int32, pin_memory=True) for _ in range(2)]
        self._req_done = [None, None]
        self._req_i = 0
        self.n_req = 0
        self.route_class = (self.decode_launched, self.prefill_launched)
        self._graph = None
        self._graph_class = None
        self._graph_io = None
        self.recaptures = 0
        self.table = SegmentTable(
            perm=torch.zeros(self.max_tokens, dtype=torch.int32, device=dev),
            seg_off=torch.zeros(self.max_requests + 1, dtype=torch.int32, device=dev),
            seg_slot=torch.zeros(self.max_requests, dtype=torch.int32, device=dev),
            seg_rank=torch.zeros(self.max_requests, dtype=torch.int32, device=dev),
            n_seg=torch.zeros(1, dtype=torch.int32, device=dev),
            n_tokens=self.max_tokens,
        )

    # -- host side ------------------------------------------------------------------------
    def upload(self, req_slot, req_rank, req_ntok, stream=None) -> int:
        """Stage the batch's request arrays in pinned memory and copy them asynchronously.
        Returns the number of tokens of the batch."""
        n = len(req_slot)
        if n > self.max_requests:
            raise ValueError(f"{n} requests > max_requests {self.max_requests}")
        ntok = np.asarray(req_ntok, dtype=np.int64)
        total = int(ntok.sum())
        if total > self.max_tokens:
            raise ValueError(f"{total} tokens > max_tokens {self.max_tokens}")
        m = n if self.graph_requests is None else self.graph_requests
        if n > m:
            raise ValueError(f"{n} requests > graph_requests {m}")
        b = self._req_i
        self._req_i ^= 1
        if self._req_done[b] is not None:
            self._req_done[b].synchronize()  # this staging buffer's previous copy has been consumed
        host = self._req_host[b]
        h = host.numpy()
        h[0, :n] = req_slot
        h[1, :n] = req_rank
        h[2, :n] = req_ntok
        if m > n:  # padding requests: no adapter, no tokens
            h[0, n:m] = -1
            h[1, n:m] = 0
            h[2, n:m] = 0
        s = stream or torch.cuda.current_stream(self.pool.device)
        with torch.cuda.stream(s):
            self.req_dev[:, :m].copy_(host[:, :m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s)
        self._req_done[b] = ev
        self.n_req = m
        if self.route_hints:
            lo, hi = segment_token_bounds(req_slot, req_rank, req_ntok)
            self.pool.set_prefill_route(self.prefill_min_tokens, lo, hi)
            self.prefill_launched = self.prefill_min_tokens > 0 and hi >= self.prefill_min_tokens
            self.decode_launched = not self.prefill_launched or lo < self.prefill_min_tokens
        self.route_class = (self.decode_launched, self.prefill_launched)
        return total

    # -- device side (capturable) ------------------------------------------------------------
    def build(self, stream=None) -> SegmentTable:
        """K4 segment table + the step's launch plan (two single-CTA kernels)."""
        n = self.n_req
        build_segments(self.req_dev[0, :n], self.req_dev[1, :n], self.req_dev[2, :n], device=self.pool.device,
                       stream=stream, out=self.table)
        build_plan(self.table, pool=self.pool, stream=stream)
        return self.table

    def apply_layer(self, layer: int, xs: Sequence[torch.Tensor], ys: Sequence[torch.Tensor], stream=None,
                    last: bool = True):
        """xs[g]: input of projection group g; ys[p]: output of projection p (in place).
        With last=False the step continues with layer + 1 (same plan): the final group's apply
        prefetches that layer's first group."""
        G = len(self.proj_groups)
        for g, projs in enumerate(self.proj_groups):
            if self.l2_prefetch_bytes > 0:
                if g + 1 < G:
                    self.pool.set_next_apply(layer, self.proj_groups[g + 1])
                elif not last and layer + 1 < self.pool.n_layers:
                    self.pool.set_next_apply(layer + 1, self.proj_groups[0])
                else:
                    self.pool.set_next_apply()
            if len(projs) == 1:
                lora_apply_table(xs[g], ys[projs[0]], self.table, pool=self.pool, layer=layer, proj=projs[0],
                                 stream=stream)
            else:
                lora_apply_multi([xs[g]] * len(projs), [ys[p] for p in projs], self.table, pool=self.pool,
                                 layer=layer, projs=projs, stream=stream)

    def launches_per_step(self) -> int:
        """Kernels per step: segment builder + plan + per (layer, group) the decode kernel
        and/or the fused tcgen05 prefill kernel."""
        per = (1 if self.decode_launched else 0) + (1 if self.prefill_launched else 0)
        return 2 + self.pool.n_layers * len(self.proj_groups) * per

    def run(self, xs_per_layer, ys_per_layer, stream=None) -> None:
        """K4 + every (layer, group) apply, on `stream`."""
        self.build(stream)
        L = self.pool.n_layers
        for layer in range(L):
            self.apply_layer(layer, xs_per_layer[layer], ys_per_layer[layer], stream, last=layer + 1 == L)

    # -- CUDA-graph step (capture once, replay per step) ---------------------------------
    def capture(self, xs_per_layer, ys_per_layer, stream) -> None:
        """Capture `run` (K4 + plan + every apply) over these activation buffers as one CUDA
        graph.  The kernel families launched (decode GEMV and/or tcgen05 prefill) follow the
        routing class of the last upload; `replay` re-captures when a later batch needs a
        family the graph does not contain, so a replay never skips segments."""
        torch.cuda.synchronize(self.pool.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            self.run(xs_per_layer, ys_per_layer)
        self._graph = g
        self._graph_class = self.route_class
        self._graph_io = (xs_per_layer, ys_per_layer, stream)

    def replay(self) -> None:
        """Replay the captured step on its stream for the batch of the last upload."""
        if self._graph is None:
            raise RuntimeError("capture() the step before replay()")
        need_dec, need_pre = self.route_class
        has_dec, has_pre = self._graph_class
        if (need_dec and not has_dec) or (need_pre and not has_pre):
            # the routing class widened (e.g. the first prefill after decode-only steps): the
            # graph would skip a kernel family, so capture one that launches both
            self.recaptures += 1
            xs, ys, stream = self._graph_io
            stream.synchronize()
            self.decode_launched = self.decode_launched or has_dec
            self.prefill_launched = self.prefill_launched or has_pre
            if self.route_hints:
                self.pool.set_prefill_route(self.prefill_min_tokens, 0 if self.decode_launched else
                                            self.prefill_min_tokens, -1 if self.prefill_launched else 0)
            self.route_class = (self.decode_launched, self.prefill_launched)
            self.capture(xs, ys, stream)
        with torch.cuda.stream(self._graph_io[2]):
            self._graph.replay()

    def check_device_error(self, stream=None) -> None:
        """Raise if any kernel of the steps so far met a device-side limit (synchronises)."""
        self.pool.check_device_error(stream=stream)
