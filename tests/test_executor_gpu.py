"""GPU parity of the exact path the bench times: LoraStepExecutor end to end.

upload (pinned H2D of the request table) -> build (K4 segment table + launch plan) -> every
(layer, projection group) apply (fused q/k/v launch + o launch, or q; k+v; o under GQA),
eager and as a captured CUDA graph replayed for several batches.  Every (layer, projection)
output is checked against the numpy oracle (oracle/lora_ref.py) — the seam this replaces is
the reference's step assembly, engine.py:443-455, and the LoRA term of
CostModel.step_duration, engine.py:67-77.

Tolerances (BASELINE.json north_star): fp32 rtol 1e-5; bf16 with fp32 accumulation rtol 2e-2
against the oracle on the same bf16-rounded inputs (absolute floor 2e-2 on O(1) outputs).
"""
from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

from oracle.lora_ref import bf16_round, lora_apply_ref
from oracle.pool_ref import unpack_block
from oracle.segments_ref import build_segments_ref

pytestmark = pytest.mark.gpu

BF16_RTOL, BF16_ATOL = 2e-2, 2e-2
FP32_RTOL, FP32_ATOL = 1e-5, 1e-5

H7B = 4096


def _fill_random(pool, slot_ranks, seed):
    """Bind slots to consecutive pages and fill every page with N(0, 0.02) device randoms."""
    from paper_2411_17741_b200.pool import pages_for_rank

    gen = torch.Generator(device=pool.device)
    gen.manual_seed(seed)
    page = 0
    for slot, r in slot_ranks.items():
        n = pages_for_rank(r)
        pool.set_slot(slot, r, list(range(page, page + n)))
        buf = (torch.randn(n * pool.page_bytes // pool.elem_bytes, generator=gen, device=pool.device) * 0.02)
        pool.fill_from_device(slot, buf.to(pool.dtype).view(torch.uint8))
        page += n
    torch.cuda.synchronize()


def _read_adapter(pool, slot, rank, layer, proj):
    """(A [h_in, r], B [r, h_out]) of one (layer, proj) read back from the pool pages
    (un-swizzled with the oracle's page-layout restatement)."""
    from paper_2411_17741_b200 import _lib

    es = pool.elem_bytes
    npdt = np.float32 if es == 4 else np.uint16
    a_off, b_off = pool.block_offsets(layer, proj)
    h_in, h_out = pool.h_in[proj], pool.h_out[proj]
    a_rows, b_rows = [], []
    for page in pool.slot_pages[slot]:
        for off, n, dst in ((a_off, h_in, a_rows), (b_off, h_out, b_rows)):
            nbytes = 8 * n * es
            host = np.empty(nbytes, dtype=np.uint8)
            _lib.call("cham_pool_copy_out", pool.handle, page * pool.page_bytes + off, nbytes,
                      host.ctypes.data_as(ctypes.c_void_p), torch.cuda.current_stream().cuda_stream)
            blk = unpack_block(host, 0, n, es, npdt)
            if es == 2:
                blk = (blk.astype(np.uint32) << 16).view(np.float32)
            dst.append(blk)
    at = np.concatenate(a_rows)[:rank]  # [r, h_in]
    b = np.concatenate(b_rows)[:rank]   # [r, h_out]
    return at.T.copy(), b.copy()


class _Model:
    """Pool + executor + capacity activation buffers for one projection layout."""

    def __init__(self, n_layers, h_in, h_out, groups, slot_ranks, dtype=torch.bfloat16, max_tokens=1024,
                 graph_requests=None, seed=0, route_hints=True):
        from paper_2411_17741_b200.executor import LoraStepExecutor
        from paper_2411_17741_b200.pool import AdapterPool, pages_for_rank

        self.dtype = dtype
        self.groups = groups
        self.slot_ranks = slot_ranks
        n_pages = sum(pages_for_rank(r) for r in slot_ranks.values())
        self.pool = AdapterPool(n_pages, n_layers, h_in, h_out, dtype=dtype, n_slots=max(slot_ranks) + 1,
                                max_tokens=max_tokens)
        _fill_random(self.pool, slot_ranks, seed)
        self.ex = LoraStepExecutor(self.pool, max_requests=1024, max_tokens=max_tokens, proj_groups=groups,
                                   graph_requests=graph_requests, route_hints=route_hints)
        dev = self.pool.device
        P = len(h_in)
        self.n_layers, self.P = n_layers, P
        self.xs = [[torch.zeros(max_tokens, h_in[g[0]], dtype=dtype, device=dev) for g in groups]
                   for _ in range(n_layers)]
        self.ys = [[torch.zeros(max_tokens, h_out[p], dtype=dtype, device=dev) for p in range(P)]
                   for _ in range(n_layers)]
        self._adapters = {}

    def adapters(self, layer, proj):
        key = (layer, proj)
        if key not in self._adapters:
            self._adapters[key] = {s: _read_adapter(self.pool, s, r, layer, proj) for s, r in self.slot_ranks.items()}
        return self._adapters[key]

    def load_batch(self, req_slot, req_ntok, seed):
        """Random activations for the batch's T rows (rows beyond T zero); uploads the table."""
        rng = np.random.default_rng(seed)
        T = int(np.sum(req_ntok))
        self.T = T
        self.x0, self.y0 = [], []
        for layer in range(self.n_layers):
            xl = []
            for g, projs in enumerate(self.groups):
                x = rng.standard_normal((T, self.xs[layer][g].shape[1])).astype(np.float32)
                x = bf16_round(x) if self.dtype == torch.bfloat16 else x
                self.xs[layer][g].zero_()
                self.xs[layer][g][:T].copy_(torch.from_numpy(x))
                xl.append(x)
            self.x0.append(xl)
            yl = []
            for p in range(self.P):
                y = rng.standard_normal((T, self.ys[layer][p].shape[1])).astype(np.float32)
                y = bf16_round(y) if self.dtype == torch.bfloat16 else y
                yl.append(y)
            self.y0.append(yl)
        self.reset_y()
        req_rank = [self.slot_ranks[s] if s >= 0 else 0 for s in req_slot]
        self.req = (list(req_slot), req_rank, list(req_ntok))
        self.ex.upload(np.asarray(req_slot, np.int32), np.asarray(req_rank, np.int32),
                       np.asarray(req_ntok, np.int32))
        torch.cuda.synchronize()

    def reset_y(self):
        for layer in range(self.n_layers):
            for p in range(self.P):
                self.ys[layer][p].zero_()
                self.ys[layer][p][:self.T].copy_(torch.from_numpy(self.y0[layer][p]))

    def check(self, layer_projs=None):
        perm, off, sl, rk = build_segments_ref(*self.req)
        # the device table must be the canonical one (bit-exact)
        dperm, doff, dsl, drk = self.ex.table.to_host()
        np.testing.assert_array_equal(dperm, perm)
        np.testing.assert_array_equal(doff, off)
        np.testing.assert_array_equal(dsl, sl)
        np.testing.assert_array_equal(drk, rk)
        g_of = {p: g for g, projs in enumerate(self.groups) for p in projs}
        todo = layer_projs or [(l, p) for l in range(self.n_layers) for p in range(self.P)]
        for layer, p in todo:
            ref = lora_apply_ref(self.x0[layer][g_of[p]], self.y0[layer][p], perm, off, sl, rk,
                                 self.adapters(layer, p))
            got = self.ys[layer][p][:self.T].float().cpu().numpy()
            if self.dtype == torch.bfloat16:
                np.testing.assert_allclose(got, bf16_round(ref.astype(np.float32)), rtol=BF16_RTOL, atol=BF16_ATOL,
                                           err_msg=f"layer {layer} proj {p}")
            else:
                np.testing.assert_allclose(got, ref, rtol=FP32_RTOL, atol=FP32_ATOL, err_msg=f"layer {layer} proj {p}")

    def close(self):
        self.pool.close()


def _decode_batch(rng, slots, n):
    return rng.choice(slots, n).tolist(), [1] * n


def _mixed_batch(rng, slots, n_dec, prefill):
    """prefill: list of (slot, tokens) — prefills first, then decoders (engine.py:443-451)."""
    ps = [s for s, _ in prefill]
    pt = [t for _, t in prefill]
    ds = rng.choice(slots, n_dec).tolist()
    return ps + ds, pt + [1] * n_dec


SLOT_RANKS = {0: 8, 1: 16, 2: 32, 3: 64, 4: 128, 5: 8, 6: 24, 7: 16, 8: 128, 9: 40, 10: 64, 11: 8}


@pytest.mark.parametrize("graph", [False, True])
def test_executor_multilayer_qkv_o_decode_and_mixed(graph):
    """4 layers x q/k/v/o (7B dims), fused q/k/v + o launches; a decode-only batch then a
    mixed prefill/decode batch through the same executor (eager or one captured graph)."""
    rng = np.random.default_rng(11)
    m = _Model(4, [H7B] * 4, [H7B] * 4, [[0, 1, 2], [3]], SLOT_RANKS, graph_requests=128 if graph else None)
    s = torch.cuda.Stream()
    slots = list(SLOT_RANKS)
    try:
        m.load_batch(*_decode_batch(rng, slots, 96), seed=1)
        with torch.cuda.stream(s):
            m.ex.run(m.xs, m.ys)  # eager (also sets the kernel attributes before any capture)
        s.synchronize()
        m.check()
        if graph:
            m.reset_y()
            m.ex.capture(m.xs, m.ys, s)
            m.ex.replay()
            s.synchronize()
            m.check()
        # a different batch: prefill segments (tcgen05 route) + decode tokens
        m.load_batch(*_mixed_batch(rng, slots, 40, [(3, 70), (4, 128), (2, 200), (9, 64)]), seed=2)
        if graph:
            m.ex.replay()  # the routing class widened: the executor re-captures instead of skipping
            assert m.ex.recaptures == 1
        else:
            with torch.cuda.stream(s):
                m.ex.run(m.xs, m.ys)
        s.synchronize()
        m.check()
        m.ex.check_device_error()
        if graph:
            # back to decode-only: the widened graph still serves it (no new capture)
            m.load_batch(*_decode_batch(rng, slots, 128), seed=3)
            m.ex.replay()
            s.synchronize()
            assert m.ex.recaptures == 1
            m.check()
    finally:
        m.close()


def test_executor_graph_prefill_first_then_decode():
    """A graph captured on an all-prefill step (no decode kernel in it) must not silently skip
    the decode tokens of a later step (the replay re-captures)."""
    rng = np.random.default_rng(12)
    m = _Model(2, [H7B] * 4, [H7B] * 4, [[0, 1, 2], [3]], SLOT_RANKS, graph_requests=64)
    s = torch.cuda.Stream()
    try:
        m.load_batch([3, 4, 1], [64, 96, 128], seed=4)
        assert m.ex.route_class == (False, True)
        with torch.cuda.stream(s):
            m.ex.run(m.xs, m.ys)
        s.synchronize()
        m.check()
        m.reset_y()
        m.ex.capture(m.xs, m.ys, s)
        m.ex.replay()
        s.synchronize()
        m.check()
        m.load_batch(*_decode_batch(rng, list(SLOT_RANKS), 50), seed=5)
        m.ex.replay()
        s.synchronize()
        assert m.ex.recaptures == 1
        m.check()
    finally:
        m.close()


def test_executor_gqa_70b_shard_dims_graph():
    """GQA layout at Llama-2-70B dims: q 8192->8192, k/v 8192->1024, o 8192->8192, groups
    q; k+v; o (the C5 TP=1 launch layout), 2 layers, graph replay over two batches."""
    rng = np.random.default_rng(13)
    sr = {0: 64, 1: 32, 2: 8, 3: 128, 4: 16}
    m = _Model(2, [8192, 8192, 8192, 8192], [8192, 1024, 1024, 8192], [[0], [1, 2], [3]], sr, graph_requests=96)
    s = torch.cuda.Stream()
    try:
        m.load_batch(*_decode_batch(rng, list(sr), 64), seed=6)
        with torch.cuda.stream(s):
            m.ex.run(m.xs, m.ys)
        s.synchronize()
        m.check()
        m.reset_y()
        m.ex.capture(m.xs, m.ys, s)
        m.ex.replay()
        s.synchronize()
        m.check()
        m.load_batch(*_mixed_batch(rng, list(sr), 30, [(0, 80), (3, 64)]), seed=7)
        m.ex.replay()
        s.synchronize()
        m.check()
    finally:
        m.close()


def test_executor_fp32_multilayer_rtol_1e5():
    """fp32 pool (decode kernel only, CUDA-core FP32 FMA): 3 layers, per-projection launches,
    multi-token segments, graph replay of a second batch."""
    rng = np.random.default_rng(14)
    sr = {0: 8, 1: 16, 2: 24, 3: 64}
    m = _Model(3, [2048] * 4, [2048] * 4, [[0], [1], [2], [3]], sr, dtype=torch.float32, graph_requests=48)
    s = torch.cuda.Stream()
    try:
        m.load_batch([0, 1, 2, 3, 0, 2] + rng.choice(4, 20).tolist(), [5, 9, 3, 17, 2, 1] + [1] * 20, seed=8)
        with torch.cuda.stream(s):
            m.ex.run(m.xs, m.ys)
        s.synchronize()
        m.check()
        m.reset_y()
        m.ex.capture(m.xs, m.ys, s)
        m.load_batch(rng.choice(4, 40).tolist(), [1] * 40, seed=9)
        m.ex.replay()
        s.synchronize()
        m.check()
    finally:
        m.close()


def test_c2_full_size_32_layers_graph():
    """The bench's C2 step itself: Llama-2-7B dims, 32 layers x q/k/v/o, the 100-adapter
    catalog, 256 decode tokens of decode_batch(seed 0), executor graph; 8 sampled
    (layer, proj) outputs (every projection, first/last layers) checked against the oracle."""
    from paper_2411_17741_b200.model import build_catalog
    from paper_2411_17741_b200.workload import decode_batch

    catalog = build_catalog(100)
    ids = list(catalog)
    batch = decode_batch(0, 256, 100)
    used = sorted(set(batch), key=ids.index)
    slot_of = {a: i for i, a in enumerate(used)}
    sr = {slot_of[a]: catalog[a].rank for a in used}
    m = _Model(32, [H7B] * 4, [H7B] * 4, [[0, 1, 2], [3]], sr, max_tokens=512, graph_requests=256, seed=1234)
    s = torch.cuda.Stream()
    try:
        m.load_batch([slot_of[a] for a in batch], [1] * 256, seed=10)
        with torch.cuda.stream(s):
            m.ex.run(m.xs, m.ys)
        s.synchronize()
        m.reset_y()
        m.ex.capture(m.xs, m.ys, s)
        for _ in range(2):  # replays are idempotent given the same inputs
            m.reset_y()
            m.ex.replay()
            s.synchronize()
        m.check([(0, 0), (0, 3), (7, 1), (12, 2), (19, 3), (25, 0), (31, 1), (31, 2)])
        m.ex.check_device_error()
    finally:
        m.close()


def test_c3_full_4096_tokens_two_layers():
    """C3 shape: 64 prefill segments x 64 tokens (prefill_batch seed 0, power-law ranks) over
    2 layers of 7B q/k/v/o — every segment on the tcgen05 path — every (layer, proj) checked."""
    from paper_2411_17741_b200.workload import prefill_batch, rank_of_id

    pids, pntok = prefill_batch(0)
    ids = list(dict.fromkeys(pids))
    slot_of = {a: i for i, a in enumerate(ids)}
    sr = {slot_of[a]: rank_of_id(a) for a in ids}
    m = _Model(2, [H7B] * 4, [H7B] * 4, [[0, 1, 2], [3]], sr, max_tokens=4096, seed=77)
    s = torch.cuda.Stream()
    try:
        m.load_batch([slot_of[a] for a in pids], pntok, seed=11)
        assert m.ex.route_class == (False, True)
        with torch.cuda.stream(s):
            m.ex.run(m.xs, m.ys)
        s.synchronize()
        m.check()
        m.ex.check_device_error()
    finally:
        m.close()


def test_prefill_stress_chained_launches_do_not_fault():
    """Soak of the tcgen05 prefill kernel at the C3 shape: 3 rounds x 1,200 PDL-chained
    launches (2 layers x (q/k/v + o) per step, 300 graph replays), each round ending with a
    synchronisation and a device-error check; then one more step is checked against the oracle.
    Before every replay a copy kernel on the same stream rewrites the first layer's x (same
    values): the serving pattern that made x loads with an L2 evict_last hint fault the
    context in nearly every run."""
    from paper_2411_17741_b200.workload import prefill_batch, rank_of_id

    pids, pntok = prefill_batch(0)
    ids = list(dict.fromkeys(pids))
    slot_of = {a: i for i, a in enumerate(ids)}
    sr = {slot_of[a]: rank_of_id(a) for a in ids}
    m = _Model(2, [H7B] * 4, [H7B] * 4, [[0, 1, 2], [3]], sr, max_tokens=4096, seed=78)
    s = torch.cuda.Stream()
    try:
        m.load_batch([slot_of[a] for a in pids], pntok, seed=12)
        with torch.cuda.stream(s):
            m.ex.run(m.xs, m.ys)
        s.synchronize()
        m.ex.capture(m.xs, m.ys, s)
        x_src = m.xs[0][0].clone()
        for _ in range(3):
            for _ in range(300):
                with torch.cuda.stream(s):
                    m.xs[0][0].copy_(x_src)
                m.ex.replay()
            s.synchronize()
            m.ex.check_device_error()
        m.reset_y()
        m.ex.replay()
        s.synchronize()
        m.check()
    finally:
        m.close()
