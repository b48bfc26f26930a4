"""C5 tensor-parallel sequencing on CPU with gloo, world_size 2.

Each rank holds its h_in shard of A and h_out shard of B, runs TensorParallelLora with the
shrink/expand operators replaced by the numpy oracle (the device kernels are covered by the
GPU tests), and the concatenated y shards must equal the unsharded oracle result.  Checks
one all-reduce per projection group (q/k/v fused), GQA-shaped k/v widths, mixed ranks,
multi-token requests and rows without an adapter.
"""
import os
import socket
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]

H_IN = [64, 64, 64, 64]
H_OUT = [64, 16, 16, 64]  # q, k, v (GQA-narrow), o
LAYERS = 2
SLOT_RANKS = {0: 8, 1: 16, 2: 24, 5: 8}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    from oracle.lora_ref import make_adapters
    from oracle.segments_ref import build_segments_ref

    rng = np.random.default_rng(11)
    adapters = {}  # (layer, proj) -> slot -> (A, B)
    for l in range(LAYERS):
        for p in range(4):
            adapters[l, p] = make_adapters(rng, SLOT_RANKS, H_IN[p], H_OUT[p])
    req_slot = [2, -1, 0, 5, 2, 1, 0]
    req_rank = [SLOT_RANKS.get(s, 0) for s in req_slot]
    req_ntok = [3, 2, 1, 1, 4, 2, 1]
    T = sum(req_ntok)
    tables = build_segments_ref(req_slot, req_rank, req_ntok)
    xs = {(l, g): rng.standard_normal((T, 64)).astype(np.float32) for l in range(LAYERS) for g in range(2)}
    ys = {(l, p): rng.standard_normal((T, H_OUT[p])).astype(np.float32) for l in range(LAYERS) for p in range(4)}
    return adapters, tables, xs, ys, T


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    from oracle.lora_ref import lora_expand_ref, lora_shrink_ref
    from paper_2411_17741_b200.tp import TensorParallelLora, shard_bounds

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    adapters, (perm, seg_off, seg_slot, seg_rank), xs, ys, T = _problem()
    local = {}
    for (l, p), per_slot in adapters.items():
        i0, i1 = shard_bounds(H_IN[p], world, rank)
        o0, o1 = shard_bounds(H_OUT[p], world, rank)
        local[l, p] = {s: (a[i0:i1], b[:, o0:o1]) for s, (a, b) in per_slot.items()}

    def shrink(x, v, slot_ids, seg_offsets, ranks, *, pool, layer, proj, perm=None, plan=None, stream=None):
        got = lora_shrink_ref(x.numpy(), perm, seg_offsets, slot_ids, ranks, local[layer, proj], v.shape[1])
        v[: got.shape[0]] = torch.from_numpy(got.astype(np.float32))

    def expand(v, y, slot_ids, seg_offsets, ranks, *, pool, layer, proj, perm=None, plan=None, stream=None):
        n = int(seg_offsets[-1])
        y[:] = torch.from_numpy(lora_expand_ref(v[:n].numpy(), y.numpy(), perm, seg_offsets, slot_ids, ranks,
                                                local[layer, proj]).astype(np.float32))

    pool = SimpleNamespace(n_proj=4, device=torch.device("cpu"))
    tp = TensorParallelLora(pool, max_tokens=T, r_stride=24, proj_groups=[[0, 1, 2], [3]], shrink=shrink,
                            expand=expand, device="cpu")
    result = {}
    for l in range(LAYERS):
        i0, i1 = shard_bounds(64, world, rank)
        x_sh = [torch.from_numpy(xs[l, g][:, i0:i1].copy()) for g in range(2)]
        y_sh = []
        for p in range(4):
            o0, o1 = shard_bounds(H_OUT[p], world, rank)
            y_sh.append(torch.from_numpy(ys[l, p][:, o0:o1].copy()))
        tp.apply_layer(l, x_sh, y_sh, seg_slot, seg_off, seg_rank, perm=perm, n_positions=int(seg_off[-1]))
        for p in range(4):
            parts = [torch.empty_like(y_sh[p]) for _ in range(world)]
            dist.all_gather(parts, y_sh[p])
            result[l, p] = torch.cat(parts, dim=1).numpy()
    if rank == 0:
        np.savez(os.path.join(out_dir, "tp.npz"), allreduces=tp.allreduce_count,
                 **{f"y_{l}_{p}": v for (l, p), v in result.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_tp2_gloo_matches_unsharded_oracle(tmp_path):
    from oracle.lora_ref import lora_apply_ref

    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "tp.npz")
    assert int(got["allreduces"]) == 2 * LAYERS  # one per projection group per layer
    adapters, (perm, seg_off, seg_slot, seg_rank), xs, ys, T = _problem()
    for l in range(LAYERS):
        for p in range(4):
            want = lora_apply_ref(xs[l, 0 if p < 3 else 1], ys[l, p], perm, seg_off, seg_slot, seg_rank,
                                  adapters[l, p])
            np.testing.assert_allclose(got[f"y_{l}_{p}"], want, rtol=1e-5, atol=1e-5)
    # the no-adapter request's rows (tokens 3, 4) are untouched
    np.testing.assert_array_equal(got["y_0_0"][3:5], ys[0, 0][3:5])


def test_shard_helpers():
    from paper_2411_17741_b200.tp import shard_adapter, shard_bounds, shard_dims

    assert shard_bounds(8192, 4, 3) == (6144, 8192)
    with pytest.raises(ValueError):
        shard_bounds(1000, 3, 0)
    assert shard_dims([8192, 8192, 8192, 8192], [8192, 1024, 1024, 8192], 8) == ([1024] * 4, [1024, 128, 128, 1024])
    a = [np.arange(16).reshape(8, 2)]
    b = [np.arange(16).reshape(2, 8)]
    a1, b1 = shard_adapter(a, b, [8], [8], 2, 1)
    assert a1[0].tolist() == a[0][4:].tolist() and b1[0].tolist() == b[0][:, 4:].tolist()
