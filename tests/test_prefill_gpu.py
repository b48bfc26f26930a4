"""GPU parity of the tcgen05 prefill path (K3, cham_prefill.cu) through the C ABI.

Segments with >= prefill_min_tokens tokens (default 64) and rank <= 128 of a bf16 pool run
on the tensor-core kernels; everything else on the decode kernel.  Each case is checked
against the numpy oracle on the same bf16-rounded inputs (rtol 2e-2, atol 2e-2 on outputs
of magnitude ~1; BASELINE.json north_star) and, where useful, against the decode-only route.
"""
import numpy as np
import pytest
import torch

from oracle.lora_ref import bf16_round, lora_apply_ref, make_adapters
from oracle.segments_ref import build_segments_ref

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-2, 2e-2


def _setup(h_in, h_out, slot_ranks, req_slots, req_ntok, seed, n_proj=1, max_tokens=4096):
    from paper_2411_17741_b200.pool import AdapterPool

    rng = np.random.default_rng(seed)
    adapters = [make_adapters(rng, slot_ranks, h_in, h_out, bf16=True) for _ in range(n_proj)]
    T = int(np.sum(req_ntok))
    x = bf16_round(rng.standard_normal((T, h_in)).astype(np.float32))
    y0 = [bf16_round(rng.standard_normal((T, h_out)).astype(np.float32)) for _ in range(n_proj)]
    npages = sum(-(-r // 8) for r in slot_ranks.values())
    pool = AdapterPool(npages, 1, [h_in] * n_proj, [h_out] * n_proj, dtype=torch.bfloat16,
                       n_slots=max(slot_ranks) + 1, max_tokens=max_tokens)
    page = 0
    for s, r in slot_ranks.items():
        npg = -(-r // 8)
        pool.set_slot(s, r, list(range(page, page + npg)))
        page += npg
        packed = pool.pack_host([torch.from_numpy(adapters[p][s][0]) for p in range(n_proj)],
                                [torch.from_numpy(adapters[p][s][1]) for p in range(n_proj)], r)
        pool.fill_async(s, packed)
    torch.cuda.synchronize()
    req_rank = [slot_ranks[s] if s >= 0 else 0 for s in req_slots]
    table = build_segments_ref(req_slots, req_rank, req_ntok)
    return pool, adapters, x, y0, table


def _apply(pool, x, y0, table, proj=0):
    from paper_2411_17741_b200.ops import lora_apply

    perm, seg_off, seg_slot, seg_rank = table
    xd = torch.from_numpy(x).to("cuda", torch.bfloat16)
    yd = torch.from_numpy(y0).to("cuda", torch.bfloat16)
    lora_apply(xd, yd, seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=proj, perm=perm)
    torch.cuda.synchronize()
    return yd.float().cpu().numpy()


def _ref(x, y0, table, adapters):
    perm, seg_off, seg_slot, seg_rank = table
    return bf16_round(lora_apply_ref(x, y0, perm, seg_off, seg_slot, seg_rank, adapters).astype(np.float32))


def test_mixed_prefill_and_decode_batch():
    """Prefill segments of 64..300 tokens (partial and multiple 128-token tiles), odd page
    counts (ranks 8, 24, 40, 72), rank 256 (decode kernel), decode requests interleaved
    with prefills of the same adapter, and rows without an adapter."""
    slot_ranks = {0: 8, 1: 24, 2: 40, 3: 72, 4: 128, 5: 256, 6: 16}
    req_slots = [1, 0, 6, 2, -1, 3, 4, 5, 6, 0, 1, 2, 3, 6, 4]
    req_ntok = [70, 129, 3, 300, 5, 64, 128, 90, 1, 1, 1, 1, 1, 1, 200]
    pool, adapters, x, y0, table = _setup(4096, 4096, slot_ranks, req_slots, req_ntok, seed=11)
    got = _apply(pool, x, y0[0], table)
    ref = _ref(x, y0[0], table, adapters[0])
    np.testing.assert_allclose(got, ref, rtol=RTOL, atol=ATOL)
    # decode-only route gives the same answer
    pool.set_prefill_route(0)
    got_dec = _apply(pool, x, y0[0], table)
    np.testing.assert_allclose(got_dec, ref, rtol=RTOL, atol=ATOL)
    pool.close()


def test_single_tile_uses_split_k():
    """One 100-token segment: one tile, so the shrink splits K 8 ways (partials summed in
    the expand kernel)."""
    slot_ranks = {0: 64}
    pool, adapters, x, y0, table = _setup(4096, 4096, slot_ranks, [0], [100], seed=12)
    got = _apply(pool, x, y0[0], table)
    np.testing.assert_allclose(got, _ref(x, y0[0], table, adapters[0]), rtol=RTOL, atol=ATOL)
    pool.close()


@pytest.mark.parametrize("h_in,h_out", [(8192, 1024), (1024, 2048), (2048, 8192)])
def test_rectangular_projections(h_in, h_out):
    slot_ranks = {0: 64, 1: 32, 2: 8}
    pool, adapters, x, y0, table = _setup(h_in, h_out, slot_ranks, [0, 1, 2, 1], [130, 64, 65, 2], seed=13)
    got = _apply(pool, x, y0[0], table)
    np.testing.assert_allclose(got, _ref(x, y0[0], table, adapters[0]), rtol=RTOL, atol=ATOL)
    pool.close()


def test_qkv_multi_job_launch_and_route_hints():
    """Three projections sharing x in one launch through a device segment table; then the
    same with the host hint that every segment is prefill-sized (decode kernel skipped)."""
    from paper_2411_17741_b200.ops import build_segments, lora_apply_multi

    slot_ranks = {0: 16, 1: 128, 2: 32}
    req_slots, req_ntok = [0, 1, 2, 0], [96, 200, 64, 40]
    pool, adapters, x, y0, table = _setup(4096, 4096, slot_ranks, req_slots, req_ntok, seed=14, n_proj=3)
    req_rank = [slot_ranks[s] for s in req_slots]
    refs = [_ref(x, y0[p], table, adapters[p]) for p in range(3)]
    for hint in (None, (64, 1 << 20)):
        if hint is not None:
            pool.set_prefill_route(64, *hint)
        dt = build_segments(req_slots, req_rank, req_ntok, device=pool.device)
        xd = torch.from_numpy(x).to("cuda", torch.bfloat16)
        ys = [torch.from_numpy(y).to("cuda", torch.bfloat16) for y in y0]
        lora_apply_multi([xd] * 3, ys, dt, pool=pool, layer=0, projs=[0, 1, 2])
        torch.cuda.synchronize()
        for p in range(3):
            np.testing.assert_allclose(ys[p].float().cpu().numpy(), refs[p], rtol=RTOL, atol=ATOL)
    pool.close()


def test_tp_halves_on_prefill_segments():
    """cham_lora_shrink / cham_lora_expand route prefill segments to the tcgen05 kernels
    (final fp32 v in [position][v_stride]); shrink -> expand equals the fused apply."""
    from paper_2411_17741_b200.ops import lora_expand, lora_shrink

    slot_ranks = {0: 64, 1: 8}
    req_slots, req_ntok = [0, 1, 0], [150, 70, 1]
    pool, adapters, x, y0, table = _setup(4096, 4096, slot_ranks, req_slots, req_ntok, seed=15)
    perm, seg_off, seg_slot, seg_rank = table
    xd = torch.from_numpy(x).to("cuda", torch.bfloat16)
    yd = torch.from_numpy(y0[0]).to("cuda", torch.bfloat16)
    v = torch.zeros(len(perm), 64, dtype=torch.float32, device="cuda")
    lora_shrink(xd, v, seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=0, perm=perm)
    lora_expand(v, yd, seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=0, perm=perm)
    torch.cuda.synchronize()
    np.testing.assert_allclose(yd.float().cpu().numpy(), _ref(x, y0[0], table, adapters[0]), rtol=RTOL, atol=ATOL)
    pool.close()


def test_multi_job_distinct_inputs_and_gathered_rows():
    """Jobs with different x tensors (no shared x stage) and segments whose rows are not
    contiguous in x (two requests of one adapter interleaved with others: TMA row gathers),
    tiles of 33..128 rows, ranks with odd page counts."""
    from paper_2411_17741_b200.ops import build_segments, lora_apply_multi

    slot_ranks = {0: 40, 1: 8, 2: 128, 3: 24}
    req_slots = [0, 1, 0, 2, 3, 1]
    req_ntok = [40, 70, 33, 97, 64, 9]
    pool, adapters, x, y0, table = _setup(2048, 4096, slot_ranks, req_slots, req_ntok, seed=16, n_proj=2)
    rng = np.random.default_rng(17)
    x2 = bf16_round(rng.standard_normal(x.shape).astype(np.float32))
    perm, seg_off, seg_slot, seg_rank = table
    refs = [_ref(x, y0[0], table, adapters[0]), _ref(x2, y0[1], table, adapters[1])]
    req_rank = [slot_ranks[s] for s in req_slots]
    dt = build_segments(req_slots, req_rank, req_ntok, device=pool.device)
    xs = [torch.from_numpy(v).to("cuda", torch.bfloat16) for v in (x, x2)]
    ys = [torch.from_numpy(y).to("cuda", torch.bfloat16) for y in y0]
    lora_apply_multi(xs, ys, dt, pool=pool, layer=0, projs=[0, 1])
    torch.cuda.synchronize()
    for p in range(2):
        np.testing.assert_allclose(ys[p].float().cpu().numpy(), refs[p], rtol=RTOL, atol=ATOL)
    pool.close()


def test_repeated_launches_reuse_workspaces():
    """Many back-to-back prefill applies (PDL-chained, counter parity sets and tile flags
    reused) give the same result as one apply, applied n times."""
    from paper_2411_17741_b200.ops import lora_apply

    slot_ranks = {0: 16, 1: 64}
    pool, adapters, x, y0, table = _setup(4096, 4096, slot_ranks, [0, 1], [130, 80], seed=18)
    perm, seg_off, seg_slot, seg_rank = table
    xd = torch.from_numpy(x).to("cuda", torch.bfloat16)
    y_once = torch.from_numpy(y0[0]).to("cuda", torch.bfloat16)
    lora_apply(xd, y_once, seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=0, perm=perm)
    delta = y_once.float() - torch.from_numpy(y0[0]).cuda()
    ys = [torch.from_numpy(y0[0]).to("cuda", torch.bfloat16) for _ in range(6)]
    for i in range(6):
        lora_apply(xd, ys[i], seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=0, perm=perm)
    torch.cuda.synchronize()
    for y in ys:
        assert torch.equal(y, y_once)
    assert delta.abs().max().item() > 0
    pool.close()


@pytest.mark.parametrize("seed", [101, 102, 103, 104, 105, 106])
def test_random_mixed_batches_fuzz(seed):
    """Seeded random batches across both kernels: 1-48 requests of 1-150 tokens (segments of
    64+ tokens go to the tcgen05 kernel, the rest to the decode kernel), ranks 8-128 including
    non-multiples of 16, rectangular h_in/h_out, requests without an adapter."""
    _fuzz(seed, torch.bfloat16)


@pytest.mark.parametrize("seed", [201, 202, 203])
def test_random_batches_fuzz_fp32(seed):
    """The same random batches on an fp32 pool (decode kernel only), rtol 1e-5."""
    _fuzz(seed, torch.float32)


def _fuzz(seed, dtype):
    from oracle.lora_ref import bf16_round, lora_apply_ref, make_adapters
    from oracle.segments_ref import build_segments_ref
    from paper_2411_17741_b200.ops import lora_apply
    from paper_2411_17741_b200.pool import AdapterPool

    rng = np.random.default_rng(seed)
    h_in, h_out = int(rng.choice([256, 512, 1024])), int(rng.choice([256, 512, 1024]))
    n_slots = int(rng.integers(1, 9))
    slot_ranks = {s: int(rng.choice([8, 16, 24, 32, 40, 64, 72, 128])) for s in range(n_slots)}
    bf16 = dtype == torch.bfloat16
    adapters = make_adapters(rng, slot_ranks, h_in, h_out, bf16=bf16)
    n_req = int(rng.integers(1, 49))
    req_slots = [int(s) if rng.random() > 0.1 else -1 for s in rng.integers(0, n_slots, n_req)]
    req_ntok = [int(rng.choice([1, 1, 2, 3, 64, 70, 100, 150])) for _ in range(n_req)]
    while sum(req_ntok) > 4096:
        req_ntok.pop()
        req_slots.pop()
    req_rank = [slot_ranks[s] if s >= 0 else 0 for s in req_slots]
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(req_slots, req_rank, req_ntok)
    T = int(sum(req_ntok))
    x = rng.standard_normal((T, h_in)).astype(np.float32)
    y0 = rng.standard_normal((T, h_out)).astype(np.float32)
    if bf16:
        x, y0 = bf16_round(x), bf16_round(y0)
    pool = AdapterPool(sum(-(-r // 8) for r in slot_ranks.values()), 1, [h_in], [h_out], dtype=dtype,
                       n_slots=n_slots, max_tokens=4096)
    page = 0
    for s, r in slot_ranks.items():
        npg = -(-r // 8)
        pool.set_slot(s, r, list(range(page, page + npg)))
        page += npg
        a, b = adapters[s]
        pool.fill_async(s, pool.pack_host([torch.from_numpy(a)], [torch.from_numpy(b)], r))
    torch.cuda.synchronize()
    xd = torch.from_numpy(x).to("cuda", dtype)
    yd = torch.from_numpy(y0).to("cuda", dtype)
    lora_apply(xd, yd, seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=0, perm=perm)
    torch.cuda.synchronize()
    ref = lora_apply_ref(x, y0, perm, seg_off, seg_slot, seg_rank, adapters)
    tol = 2e-2 if bf16 else 1e-5
    np.testing.assert_allclose(yd.float().cpu().numpy(), ref, rtol=tol, atol=tol if bf16 else 1e-4)
    pool.close()


@pytest.mark.parametrize("ntok", [1, 64])
def test_chained_launches_respect_pdl_dependencies(ntok):
    """Six back-to-back applies where each one's x is the previous one's y (decode-sized and
    prefill-sized segments): consecutive launches overlap through PDL, so any read of x/y
    before griddepcontrol.wait would see stale data and break the chain."""
    from oracle.lora_ref import bf16_round, lora_apply_ref, make_adapters
    from oracle.segments_ref import build_segments_ref
    from paper_2411_17741_b200.ops import lora_apply
    from paper_2411_17741_b200.pool import AdapterPool

    rng = np.random.default_rng(300 + ntok)
    H = 512
    slot_ranks = {0: 16, 1: 64, 2: 128}
    adapters = make_adapters(rng, slot_ranks, H, H, bf16=True)
    req_slots = [0, 1, 2, 1, 0, 2] * (4 if ntok == 1 else 1)
    req_ntok = [ntok] * len(req_slots)
    req_rank = [slot_ranks[s] for s in req_slots]
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(req_slots, req_rank, req_ntok)
    T = int(sum(req_ntok))
    pool = AdapterPool(sum(-(-r // 8) for r in slot_ranks.values()), 1, [H], [H], dtype=torch.bfloat16,
                       n_slots=3, max_tokens=4096)
    page = 0
    for s, r in slot_ranks.items():
        npg = -(-r // 8)
        pool.set_slot(s, r, list(range(page, page + npg)))
        page += npg
        a, b = adapters[s]
        pool.fill_async(s, pool.pack_host([torch.from_numpy(a)], [torch.from_numpy(b)], r))
    torch.cuda.synchronize()
    bufs = [bf16_round(rng.standard_normal((T, H)).astype(np.float32) * 0.5) for _ in range(7)]
    dev = [torch.from_numpy(b).to("cuda", torch.bfloat16) for b in bufs]
    for i in range(6):  # y_{i+1} += lora(x = y_i): launch i+1 reads what launch i wrote
        lora_apply(dev[i], dev[i + 1], seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=0, perm=perm)
    torch.cuda.synchronize()
    ref = [bufs[0]]
    for i in range(6):
        ref.append(bf16_round(lora_apply_ref(ref[i], bufs[i + 1], perm, seg_off, seg_slot, seg_rank, adapters)))
    # a stale read would be O(1) wrong almost everywhere.  The split-K shrink partials are
    # summed in fp32 and the V image is rounded to bf16 once: rtol is the single apply's 2e-2,
    # the absolute floor one bf16 ulp of the chain's largest outputs (|y| up to ~16: 0.0625),
    # where an output rounded to the neighbouring bf16 value is not a numerical error
    for i in range(1, 7):
        np.testing.assert_allclose(dev[i].float().cpu().numpy(), ref[i], rtol=2e-2, atol=6.25e-2)
    pool.close()
