"""Tensor-parallel LoRA apply (70B dims, r=64, TP 2/4/8).

Sharding (PEFT layout `lora_A.weight [r, h_in]`, `lora_B.weight [h_out, r]`):
  * A_i is sharded on h_in, the same way the base column-parallel layer shards x;
  * B_i is sharded on h_out, the same way the base layer shards y.
Per (layer, projection group) every rank
  1. shrinks its x shard:  v_g[k, :r] = x_g[perm[k]] . A_i[h_in shard]  (fp32, partial sums),
  2. all-reduces v (sum) — ONE collective per group: the q/k/v projections share x, so their
     v slices sit side by side in one [T, n_proj x r_stride] buffer,
  3. expands into its y shard: y_g[perm[k]] += v[k, :r] . B_i[:, h_out shard].
This is the only exchange step of the path.  Messages are 64-192 KiB at T=256 (latency
bound), hence the fusion of the group into one all-reduce.

Data-parallel configurations (C2-C4) do not use this module: they shard requests across
replicas with no collective.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

import torch
import torch.distributed as dist

from . import ops


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Even split of n columns across `world` ranks (n must divide)."""
    if n % world:
        raise ValueError(f"dimension {n} is not divisible by the TP degree {world}")
    w = n // world
    return rank * w, (rank + 1) * w


def shard_adapter(a_list, b_list, h_in: Sequence[int], h_out: Sequence[int], world: int, rank: int):
    """Per (layer, proj) block: A [h_in, r] -> A[h_in shard, :], B [r, h_out] -> B[:, h_out shard]."""
    P = len(h_in)
    a_sh, b_sh = [], []
    for lp, (a, b) in enumerate(zip(a_list, b_list)):
        p = lp % P
        i0, i1 = shard_bounds(h_in[p], world, rank)
        o0, o1 = shard_bounds(h_out[p], world, rank)
        a_sh.append(a[i0:i1])
        b_sh.append(b[:, o0:o1])
    return a_sh, b_sh


def shard_dims(h_in: Sequence[int], h_out: Sequence[int], world: int):
    """Local (h_in, h_out) of every projection on one TP rank."""
    return ([shard_bounds(h, world, 0)[1] for h in h_in], [shard_bounds(h, world, 0)[1] for h in h_out])


class TensorParallelLora:
    """One TP rank's LoRA apply over its pool shard.

    pool:      this rank's AdapterPool, built with shard_dims(...) and filled with
               shard_adapter(...) blocks;
    r_stride:  columns reserved per projection in the fused v buffer; must be at least the
               largest padded rank (multiple of 8) of any slot;
    group:     torch.distributed process group of the TP ranks (NCCL on the GPUs);
    shrink/expand: the device operators (ops.lora_shrink / ops.lora_expand); injectable so
               the host sequencing can be exercised by CPU tests.
    """

    def __init__(self, pool, max_tokens: int, r_stride: int = 64, proj_groups=None, group=None,
                 shrink: Optional[Callable] = None, expand: Optional[Callable] = None, device=None):
        if r_stride % 8:
            raise ValueError("r_stride must be a multiple of 8 (one pool page = 8 rank rows)")
        self.pool = pool
        self.r_stride = int(r_stride)
        self.proj_groups = [list(g) for g in (proj_groups or [[p] for p in range(pool.n_proj)])]
        self.group = group
        self.shrink = shrink or ops.lora_shrink
        self.expand = expand or ops.lora_expand
        # the device operators also come as multi-projection launches (one shrink for the
        # whole group, one expand per run of projections sharing h_out)
        self.multi = shrink is None and expand is None
        width = max(len(g) for g in self.proj_groups) * self.r_stride
        dev = device if device is not None else pool.device
        # flat storage: each group's operand is a CONTIGUOUS [n_pos, len(group) * r_stride] view
        self.v = torch.zeros(int(max_tokens) * width, dtype=torch.float32, device=dev)
        self.allreduce_count = 0

    def _world(self) -> int:
        if self.group is False or not dist.is_initialized():
            return 1
        return dist.get_world_size(self.group)

    def _check_ranks(self, seg_rank) -> None:
        if seg_rank is None or len(seg_rank) == 0:
            return
        rmax = int(max(int(r) for r in (seg_rank.tolist() if hasattr(seg_rank, "tolist") else seg_rank)))
        if -(-rmax // 8) * 8 > self.r_stride:
            raise ValueError(f"rank {rmax} exceeds r_stride {self.r_stride}")

    def apply_group(self, layer: int, projs: Sequence[int], x: torch.Tensor, ys: Sequence[torch.Tensor],
                    slot_ids, seg_offsets, ranks, *, perm=None, n_positions: Optional[int] = None,
                    plan=None, stream=None) -> None:
        """x: this rank's x shard [T, h_in/tp] (shared by projs); ys[i]: y shard of projs[i]."""
        T = x.shape[0]
        if self.multi and self._world() == 1:
            # TP degree 1: no exchange step, so the fused apply (shrink and expand in one
            # launch per run of projections sharing h_out) replaces the two halves
            i = 0
            while i < len(projs):
                j = i + 1
                while j < len(projs) and self.pool.h_out[projs[j]] == self.pool.h_out[projs[i]]:
                    j += 1
                ops.lora_apply_multi_arrays([x] * (j - i), list(ys[i:j]), slot_ids, seg_offsets, ranks,
                                            pool=self.pool, layer=layer, projs=list(projs[i:j]), perm=perm,
                                            plan=plan, stream=stream)
                i = j
            return
        n_pos = T if n_positions is None else int(n_positions)
        R = self.r_stride
        v = self.v[: n_pos * len(projs) * R].view(n_pos, len(projs) * R)
        tables = dict(pool=self.pool, layer=layer, perm=perm, plan=plan, stream=stream)
        if self.multi and len(projs) > 1 and len({self.pool.h_in[p] for p in projs}) == 1:
            ops.lora_shrink_multi([x] * len(projs), v, slot_ids, seg_offsets, ranks, projs=list(projs), **tables)
        else:
            for i, p in enumerate(projs):
                self.shrink(x, v[:, i * R:(i + 1) * R], slot_ids, seg_offsets, ranks, proj=p, **tables)
        if self.group is not False and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            if stream is not None:
                with torch.cuda.stream(stream):
                    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=self.group)
            else:
                dist.all_reduce(v, op=dist.ReduceOp.SUM, group=self.group)
            self.allreduce_count += 1
        i = 0
        while i < len(projs):
            j = i + 1
            if self.multi:  # the run of projections from i sharing h_out
                while j < len(projs) and self.pool.h_out[projs[j]] == self.pool.h_out[projs[i]]:
                    j += 1
            if j - i > 1:
                ops.lora_expand_multi(v[:, i * R:j * R], list(ys[i:j]), slot_ids, seg_offsets, ranks,
                                      projs=list(projs[i:j]), **tables)
            else:
                self.expand(v[:, i * R:(i + 1) * R], ys[i], slot_ids, seg_offsets, ranks, proj=projs[i], **tables)
            i = j

    def apply_layer(self, layer: int, xs: Sequence[torch.Tensor], ys: Sequence[torch.Tensor], slot_ids,
                    seg_offsets, ranks, **kw) -> None:
        """xs[g]: x shard of group g; ys[p]: y shard of projection p."""
        self._check_ranks(ranks)
        for g, projs in enumerate(self.proj_groups):
            self.apply_group(layer, projs, xs[g], [ys[p] for p in projs], slot_ids, seg_offsets, ranks, **kw)
