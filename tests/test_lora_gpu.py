"""GPU parity: the fused decode kernel (K1+K2) through the C ABI vs the numpy oracle.

Tolerances (BASELINE.json north_star): fp32 rtol 1e-5; bf16 with fp32 accumulation rtol 2e-2
against the oracle run on the same bf16-rounded inputs.  A non-zero base y0 keeps relative
errors well-posed; the absolute floor is stated per test.
"""
import numpy as np
import pytest
import torch

from oracle.lora_ref import bf16_round, lora_apply_ref, lora_expand_ref, lora_shrink_ref, make_adapters
from oracle.segments_ref import build_segments_ref

pytestmark = pytest.mark.gpu

FP32_RTOL, FP32_ATOL = 1e-5, 1e-5
BF16_RTOL, BF16_ATOL = 2e-2, 2e-2


def _pool(n_layers, h_in, h_out, dtype, n_pages, n_slots=64, max_tokens=4096):
    from paper_2411_17741_b200.pool import AdapterPool

    return AdapterPool(n_pages, n_layers, h_in, h_out, dtype=dtype, n_slots=n_slots, max_tokens=max_tokens)


def _install(pool, adapters_lp, slot_ranks, device_pack=False):
    """adapters_lp: slot -> list over (l,p) of (A, B) numpy arrays.  Binds pages in order."""
    next_page = 0
    for slot, r in slot_ranks.items():
        npg = -(-r // 8)
        pages = list(range(next_page, next_page + npg))
        next_page += npg
        pool.set_slot(slot, r, pages)
        a_list = [torch.from_numpy(a) for a, _ in adapters_lp[slot]]
        b_list = [torch.from_numpy(b) for _, b in adapters_lp[slot]]
        if device_pack:
            packed = pool.pack_device(a_list, b_list, r)
            pool.fill_from_device(slot, packed)
        else:
            packed = pool.pack_host(a_list, b_list, r)
            pool.fill_async(slot, packed)
    torch.cuda.synchronize()


def _run_case(dtype, h_in, h_out, slot_ranks, req_slots, req_ntok, seed=0, device_pack=False, perm_identity=False):
    rng = np.random.default_rng(seed)
    bf16 = dtype == torch.bfloat16
    adapters = make_adapters(rng, slot_ranks, h_in, h_out, bf16=bf16)
    T = int(np.sum(req_ntok))
    x = rng.standard_normal((T, h_in)).astype(np.float32)
    y0 = rng.standard_normal((T, h_out)).astype(np.float32)
    if bf16:
        x, y0 = bf16_round(x), bf16_round(y0)
    npages = sum(-(-r // 8) for r in slot_ranks.values())
    pool = _pool(1, [h_in], [h_out], dtype, npages)
    _install(pool, {s: [adapters[s]] for s in slot_ranks}, slot_ranks, device_pack=device_pack)
    req_rank = [slot_ranks[s] if s >= 0 else 0 for s in req_slots]
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(req_slots, req_rank, req_ntok)
    from paper_2411_17741_b200.ops import lora_apply

    xd = torch.from_numpy(x).to("cuda", dtype)
    yd = torch.from_numpy(y0).to("cuda", dtype)
    lora_apply(xd, yd, seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=0,
               perm=None if perm_identity else perm)
    torch.cuda.synchronize()
    got = yd.float().cpu().numpy()
    ref = lora_apply_ref(x, y0, None if perm_identity else perm, seg_off, seg_slot, seg_rank, adapters)
    pool.close()
    return got, ref


def _c1_batch():
    # 4 adapters ranks [8, 8, 16, 16], 32 requests, rng(0).integers(0, 4, 32)
    slots = np.random.default_rng(0).integers(0, 4, 32).tolist()
    return {0: 8, 1: 8, 2: 16, 3: 16}, slots


def test_c1_fp32_decode_rtol_1e5():
    slot_ranks, slots = _c1_batch()
    got, ref = _run_case(torch.float32, 4096, 4096, slot_ranks, slots, [1] * 32)
    np.testing.assert_allclose(got, ref, rtol=FP32_RTOL, atol=FP32_ATOL)


def test_c1_fp32_device_pack_matches_host_pack():
    slot_ranks, slots = _c1_batch()
    got, ref = _run_case(torch.float32, 4096, 4096, slot_ranks, slots, [1] * 32, device_pack=True)
    np.testing.assert_allclose(got, ref, rtol=FP32_RTOL, atol=FP32_ATOL)


@pytest.mark.parametrize("ranks", [(8, 16, 32, 64, 128), (24, 40, 128, 256)])
def test_bf16_mixed_ranks(ranks):
    rng = np.random.default_rng(1)
    slot_ranks = {i: r for i, r in enumerate(ranks)}
    slots = rng.integers(0, len(ranks), 96).tolist()
    got, ref = _run_case(torch.bfloat16, 4096, 4096, slot_ranks, slots, [1] * 96, seed=1)
    np.testing.assert_allclose(got, bf16_round(ref.astype(np.float32)), rtol=BF16_RTOL, atol=BF16_ATOL)


def test_bf16_multitoken_segments_and_no_adapter_rows():
    # prefill-like requests (several tokens) and requests without an adapter (slot -1)
    slot_ranks = {3: 16, 7: 64, 9: 8}
    slots = [3, -1, 7, 9, 3, 7, -1, 9]
    ntok = [5, 3, 9, 1, 2, 7, 4, 13]
    got, ref = _run_case(torch.bfloat16, 4096, 4096, slot_ranks, slots, ntok, seed=2)
    np.testing.assert_allclose(got, bf16_round(ref.astype(np.float32)), rtol=BF16_RTOL, atol=BF16_ATOL)


def test_bf16_gqa_shapes_70b_kv():
    # Llama-2-70B k/v projection: 8192 -> 1024 (C5 dims), rank 64
    slot_ranks = {0: 64, 1: 32}
    slots = [0, 1] * 20
    got, ref = _run_case(torch.bfloat16, 8192, 1024, slot_ranks, slots, [1] * 40, seed=3)
    np.testing.assert_allclose(got, bf16_round(ref.astype(np.float32)), rtol=BF16_RTOL, atol=BF16_ATOL)


def test_fp32_rectangular_and_identity_perm():
    slot_ranks = {0: 16}
    got, ref = _run_case(torch.float32, 2048, 1024, slot_ranks, [0] * 7, [1] * 7, seed=4, perm_identity=True)
    np.testing.assert_allclose(got, ref, rtol=FP32_RTOL, atol=FP32_ATOL)


def test_empty_batch_is_noop():
    from paper_2411_17741_b200.ops import lora_apply

    pool = _pool(1, [4096], [4096], torch.bfloat16, 1)
    x = torch.zeros(0, 4096, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(0, 4096, dtype=torch.bfloat16, device="cuda")
    lora_apply(x, y, [], [0], [], pool=pool, layer=0, proj=0)
    torch.cuda.synchronize()
    pool.close()


def test_repeated_launches_reset_workspace():
    """The persistent kernel resets its counters itself: back-to-back launches stay exact."""
    slot_ranks, slots = _c1_batch()
    rng = np.random.default_rng(5)
    adapters = make_adapters(rng, slot_ranks, 4096, 4096)
    x = rng.standard_normal((32, 4096)).astype(np.float32)
    y0 = rng.standard_normal((32, 4096)).astype(np.float32)
    pool = _pool(1, [4096], [4096], torch.float32, 6)
    _install(pool, {s: [adapters[s]] for s in slot_ranks}, slot_ranks)
    req_rank = [slot_ranks[s] for s in slots]
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(slots, req_rank, [1] * 32)
    from paper_2411_17741_b200.ops import lora_apply

    xd = torch.from_numpy(x).cuda()
    yd = torch.from_numpy(y0).cuda()
    for _ in range(5):
        lora_apply(xd, yd, seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=0, perm=perm)
    torch.cuda.synchronize()
    ref = y0.astype(np.float64)
    for _ in range(5):
        ref = lora_apply_ref(x, ref, perm, seg_off, seg_slot, seg_rank, adapters)
    np.testing.assert_allclose(yd.cpu().numpy(), ref, rtol=1e-5, atol=5e-5)
    pool.close()


def test_shrink_expand_halves_match_fused():
    slot_ranks = {0: 8, 1: 64, 2: 128}
    rng = np.random.default_rng(6)
    slots = rng.integers(0, 3, 40).tolist()
    adapters = make_adapters(rng, slot_ranks, 4096, 4096)
    x = rng.standard_normal((40, 4096)).astype(np.float32)
    y0 = rng.standard_normal((40, 4096)).astype(np.float32)
    pool = _pool(1, [4096], [4096], torch.float32, 25)
    _install(pool, {s: [adapters[s]] for s in slot_ranks}, slot_ranks)
    req_rank = [slot_ranks[s] for s in slots]
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(slots, req_rank, [1] * 40)
    from paper_2411_17741_b200.ops import lora_expand, lora_shrink

    xd = torch.from_numpy(x).cuda()
    v = torch.zeros(40, 128, dtype=torch.float32, device="cuda")
    lora_shrink(xd, v, seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=0, perm=perm)
    torch.cuda.synchronize()
    v_ref = lora_shrink_ref(x, perm, seg_off, seg_slot, seg_rank, adapters, 128)
    np.testing.assert_allclose(v.cpu().numpy(), v_ref, rtol=1e-5, atol=1e-5)
    yd = torch.from_numpy(y0).cuda()
    lora_expand(v, yd, seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=0, perm=perm)
    torch.cuda.synchronize()
    ref = lora_expand_ref(v_ref, y0, perm, seg_off, seg_slot, seg_rank, adapters)
    np.testing.assert_allclose(yd.cpu().numpy(), ref, rtol=1e-5, atol=1e-5)
    pool.close()


def test_device_segment_builder_bit_exact():
    from paper_2411_17741_b200.ops import build_segments

    rng = np.random.default_rng(7)
    # (requests, slots, most tokens per request): the sort covers only the bits of the
    # largest slot + 1, so cover no-adapter-only batches, one slot, and slots near 2^20
    for n_req, n_slots, mt in [(1, 1, 6), (256, 82, 6), (4096, 1000, 6), (333, 7, 6), (64, 64, 6), (50, 0, 6),
                               (300, 1 << 20, 200), (4096, 2, 16), (17, 255, 3), (600, 256, 3)]:
        slots = rng.integers(-1, n_slots, n_req)
        ranks = rng.choice([8, 16, 32, 64, 128], n_req)
        ntok = rng.integers(1, mt, n_req)
        tbl = build_segments(slots, ranks, ntok)
        torch.cuda.synchronize()
        got = tbl.to_host()
        want = build_segments_ref(slots, ranks, ntok)
        for g, w in zip(got, want):
            np.testing.assert_array_equal(g, w)


def test_prebuilt_plan_matches_in_kernel_plan():
    """The step-level plan (cham_build_plan) gives bit-identical results to the kernels'
    own plan construction, including multi-projection launches."""
    from paper_2411_17741_b200.ops import build_plan, build_segments, lora_apply_multi, lora_apply_table

    rng = np.random.default_rng(8)
    slot_ranks = {0: 8, 1: 16, 2: 32, 3: 64, 4: 128}
    adapters = make_adapters(rng, slot_ranks, 4096, 4096, bf16=True)
    pool = _pool(1, [4096] * 3, [4096] * 3, torch.bfloat16, 2 * sum(-(-r // 8) for r in slot_ranks.values()))
    page = 0
    for s, r in slot_ranks.items():
        n = -(-r // 8)
        pool.set_slot(s, r, list(range(page, page + n)))
        page += n
        a, b = adapters[s]
        at, bt = torch.from_numpy(a), torch.from_numpy(b)
        pool.fill_async(s, pool.pack_host([at, at * 0.5, at * 2], [bt, bt, bt * 0.25], r))
    torch.cuda.synchronize()
    slots = rng.integers(0, 5, 200)
    ntok = rng.integers(1, 4, 200)
    tbl = build_segments(slots, [slot_ranks[int(s)] for s in slots], ntok)
    T = int(ntok.sum())
    x = torch.from_numpy(bf16_round(rng.standard_normal((T, 4096)).astype(np.float32))).cuda().to(torch.bfloat16)
    ys0 = [torch.from_numpy(bf16_round(rng.standard_normal((T, 4096)).astype(np.float32))).cuda().to(torch.bfloat16)
           for _ in range(3)]
    ya = [y.clone() for y in ys0]
    lora_apply_multi([x] * 3, ya, tbl, pool=pool, layer=0, projs=[0, 1, 2])
    yb = [y.clone() for y in ys0]
    build_plan(tbl, pool=pool)
    lora_apply_multi([x] * 3, yb, tbl, pool=pool, layer=0, projs=[0, 1, 2])
    yc = ys0[1].clone()
    lora_apply_table(x, yc, tbl, pool=pool, layer=0, proj=1)
    torch.cuda.synchronize()
    for a_, b_ in zip(ya, yb):
        assert torch.equal(a_, b_)
    assert torch.equal(yb[1], yc)
    pool.close()


def test_tp2_70b_shards_through_strided_v():
    """C5 at 70B dims, TP=2 emulated on one GPU: each rank's pool holds its shard (A on h_in,
    B on h_out); shrink writes column slices of one fused q/k [n_pos, 2R] buffer, the
    all-reduce is the sum of the two ranks' buffers, expand reads the slices back.  The
    concatenated y shards must equal the unsharded oracle."""
    from paper_2411_17741_b200.ops import lora_expand, lora_shrink
    from paper_2411_17741_b200.tp import shard_bounds

    rng = np.random.default_rng(5)
    H_IN, H_OUT = [8192, 8192], [8192, 1024]  # q, k (GQA)
    slot_ranks = {0: 64, 1: 64, 2: 64}
    full = [make_adapters(rng, slot_ranks, H_IN[p], H_OUT[p], bf16=True) for p in range(2)]
    req_slots = rng.integers(0, 3, 48).tolist()
    req_slots[5] = -1
    req_rank = [64 if s >= 0 else 0 for s in req_slots]
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(req_slots, req_rank, [1] * 48)
    x = bf16_round(rng.standard_normal((48, 8192)).astype(np.float32))
    ys = [bf16_round(rng.standard_normal((48, H_OUT[p])).astype(np.float32)) for p in range(2)]
    R, world = 64, 2
    n_pos = int(seg_off[-1])
    vs, pools, yd = [], [], []
    for rank in range(world):
        i0, i1 = shard_bounds(8192, world, rank)
        h_out_l = [h // world for h in H_OUT]
        pool = _pool(1, [4096, 4096], h_out_l, torch.bfloat16, 3 * 8)
        sh = {}
        for s in slot_ranks:
            sh[s] = []
            for p in range(2):
                o0, o1 = shard_bounds(H_OUT[p], world, rank)
                a, b = full[p][s]
                sh[s].append((np.ascontiguousarray(a[i0:i1]), np.ascontiguousarray(b[:, o0:o1])))
        _install(pool, sh, slot_ranks)
        xd = torch.from_numpy(x[:, i0:i1].copy()).to("cuda", torch.bfloat16)
        v = torch.zeros(n_pos, 2 * R, dtype=torch.float32, device="cuda")
        for p in range(2):
            lora_shrink(xd, v[:, p * R:(p + 1) * R], seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=p,
                        perm=perm)
        vs.append(v)
        pools.append(pool)
        yd.append([torch.from_numpy(ys[p][:, shard_bounds(H_OUT[p], world, rank)[0]:
                                            shard_bounds(H_OUT[p], world, rank)[1]].copy()).to("cuda", torch.bfloat16)
                   for p in range(2)])
    v_sum = vs[0] + vs[1]  # the all-reduce
    for rank in range(world):
        for p in range(2):
            lora_expand(v_sum[:, p * R:(p + 1) * R], yd[rank][p], seg_slot, seg_off, seg_rank, pool=pools[rank],
                        layer=0, proj=p, perm=perm)
    torch.cuda.synchronize()
    for p in range(2):
        got = torch.cat([yd[r][p] for r in range(world)], dim=1).float().cpu().numpy()
        ref = lora_apply_ref(x, ys[p], perm, seg_off, seg_slot, seg_rank, full[p])
        np.testing.assert_allclose(got, ref, rtol=BF16_RTOL, atol=BF16_ATOL)
    for pool in pools:
        pool.close()


def test_c3_prefill_shape_bf16():
    """C3 shape at one (layer, proj): 64 segments x 64 tokens, 64 distinct adapters with
    ranks from workload.prefill_batch(0)."""
    from paper_2411_17741_b200.workload import prefill_batch, rank_of_id

    ids, ntok = prefill_batch(0)
    slot_ranks = {i: rank_of_id(a) for i, a in enumerate(ids)}
    got, ref = _run_case(torch.bfloat16, 4096, 4096, slot_ranks, list(range(64)), ntok, seed=9)
    np.testing.assert_allclose(got, ref, rtol=BF16_RTOL, atol=BF16_ATOL)


def test_paged_cache_fills_evictions_and_page_reuse():
    """Miniature C4: a Zipf stream through PagedAdapterCache with capacity for a fraction of
    the catalog.  Misses evict, pages are reused, fills run on the side stream; every step's
    lora_apply must match the oracle over the true adapter weights."""
    from paper_2411_17741_b200.adapter_cache import PagedAdapterCache
    from paper_2411_17741_b200.model import CacheConfig, make_adapter_spec
    from paper_2411_17741_b200.ops import lora_apply
    from paper_2411_17741_b200.pool import AdapterPool

    rng = np.random.default_rng(21)
    H = 256
    ranks = [8, 16, 32, 64, 128]
    catalog = {f"r{ranks[i % 5]}-{i // 5}": make_adapter_spec(f"r{ranks[i % 5]}-{i // 5}", ranks[i % 5])
               for i in range(25)}
    ids = list(catalog)
    weights = make_adapters(rng, {i: catalog[a].rank for i, a in enumerate(ids)}, H, H, bf16=True)
    pool = AdapterPool(64, 1, [H], [H], dtype=torch.bfloat16, n_slots=len(ids), max_tokens=256)
    store = {a: pool.pack_host([torch.from_numpy(weights[i][0])], [torch.from_numpy(weights[i][1])],
                               catalog[a].rank) for i, a in enumerate(ids)}
    cache = PagedAdapterCache(CacheConfig(), catalog, pool, host_store=store)
    cache.set_capacity(64 * 32, set(), 0)  # 41% of the catalog's 4,960 tokens
    p = np.array([(i + 1) ** -0.7 for i in range(len(ids))])
    p /= p.sum()
    now, evictions = 0, 0
    for step in range(40):
        now += 1000
        batch = [ids[int(k)] for k in rng.choice(len(ids), 24, p=p)]
        distinct = sorted(set(batch), key=batch.index)[:3]  # <= 1,536 pinned tokens
        batch = [a for a in batch if a in distinct]
        for a in distinct:
            if not cache.acquire(a, now).hit:
                e = cache.lookup(a)
                if not e.loading:
                    evictions += len(cache.evict_until(e.size_tokens, set(distinct), now))
                    cache.begin_load(a, now)
                cache.wait_ready([a])
                torch.cuda.current_stream().synchronize()
                cache.finish_load(a, now)
                cache.take_ref(a, now)
        slots = [cache.slot_of(a) for a in batch]
        rks = [catalog[a].rank for a in batch]
        perm, seg_off, seg_slot, seg_rank = build_segments_ref(slots, rks, [1] * len(batch))
        x = bf16_round(rng.standard_normal((len(batch), H)).astype(np.float32))
        y0 = bf16_round(rng.standard_normal((len(batch), H)).astype(np.float32))
        yd = torch.from_numpy(y0).to("cuda", torch.bfloat16)
        lora_apply(torch.from_numpy(x).to("cuda", torch.bfloat16), yd, seg_slot, seg_off, seg_rank, pool=pool,
                   layer=0, proj=0, perm=perm)
        torch.cuda.synchronize()
        ref = lora_apply_ref(x, y0, perm, seg_off, seg_slot, seg_rank, weights)
        np.testing.assert_allclose(yd.float().cpu().numpy(), ref, rtol=BF16_RTOL, atol=BF16_ATOL)
        for a in distinct:
            cache.release(a, now)
    assert evictions > 0 and cache.fill_count > len(set(ids)) // 2
    assert cache.used_tokens == cache.resident_tokens_recount()
    pool.close()


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_page_half_split_expand_units(dtype):
    """Adapters with more than 8 pages (ranks 72, 128, 256) have their expand units split
    into two page halves (half 0 leaves an fp32 partial, half 1 combines it with y); multi-
    token tiles, odd page counts and a 8192-wide output (8 column chunks) included."""
    slot_ranks = {0: 72, 1: 128, 2: 256, 3: 8}
    req_slots = [0, 1, 2, 1, 3, 0, 1, 2, 2, 1]
    req_ntok = [1, 3, 2, 1, 1, 5, 2, 1, 4, 1]
    got, ref = _run_case(dtype, 1024, 8192, slot_ranks, req_slots, req_ntok, seed=31)
    if dtype == torch.float32:
        np.testing.assert_allclose(got, ref, rtol=FP32_RTOL, atol=1e-5)
    else:
        np.testing.assert_allclose(got, ref, rtol=BF16_RTOL, atol=BF16_ATOL)


@pytest.mark.parametrize("ntok", ["decode", "mixed"])
def test_tp2_multi_projection_halves(ntok):
    """The TP halves as multi-projection launches (cham_lora_shrink_multi / _expand_multi):
    q/k/v (k/v GQA-narrow) shrink into ONE fused [n_pos, 3R] v per rank, the emulated
    all-reduce sums the two ranks' buffers, expand runs q alone and k+v in one launch.  The
    concatenated y shards must equal the unsharded oracle.  "mixed" adds a 96-token segment,
    which routes through the prefill kernel (one launch per projection there)."""
    from paper_2411_17741_b200.ops import lora_expand, lora_expand_multi, lora_shrink_multi
    from paper_2411_17741_b200.tp import shard_bounds

    rng = np.random.default_rng(12)
    H_IN, H_OUT = [2048, 2048, 2048], [2048, 256, 256]
    slot_ranks = {0: 64, 1: 40, 2: 16, 3: 64}
    full = [make_adapters(rng, slot_ranks, H_IN[p], H_OUT[p], bf16=True) for p in range(3)]
    n_req = 40
    req_slots = rng.integers(0, 4, n_req).tolist()
    req_ntok = [1] * n_req if ntok == "decode" else [1] * (n_req - 1) + [96]
    req_rank = [slot_ranks[s] for s in req_slots]
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(req_slots, req_rank, req_ntok)
    T = int(sum(req_ntok))
    x = bf16_round(rng.standard_normal((T, 2048)).astype(np.float32))
    ys = [bf16_round(rng.standard_normal((T, H_OUT[p])).astype(np.float32)) for p in range(3)]
    R, world = 64, 2
    n_pos = int(seg_off[-1])
    vs, pools, yd = [], [], []
    for rank in range(world):
        i0, i1 = shard_bounds(2048, world, rank)
        pool = _pool(1, [1024] * 3, [h // world for h in H_OUT], torch.bfloat16, 4 * 8, max_tokens=256)
        sh = {}
        for s in slot_ranks:
            sh[s] = []
            for p in range(3):
                o0, o1 = shard_bounds(H_OUT[p], world, rank)
                a, b = full[p][s]
                sh[s].append((np.ascontiguousarray(a[i0:i1]), np.ascontiguousarray(b[:, o0:o1])))
        _install(pool, sh, slot_ranks)
        xd = torch.from_numpy(x[:, i0:i1].copy()).to("cuda", torch.bfloat16)
        v = torch.full((n_pos, 3 * R), float("nan"), dtype=torch.float32, device="cuda")
        v.zero_()
        lora_shrink_multi([xd] * 3, v, seg_slot, seg_off, seg_rank, pool=pool, layer=0, projs=[0, 1, 2], perm=perm)
        vs.append(v)
        pools.append(pool)
        yd.append([torch.from_numpy(ys[p][:, shard_bounds(H_OUT[p], world, rank)[0]:
                                            shard_bounds(H_OUT[p], world, rank)[1]].copy()).to("cuda", torch.bfloat16)
                   for p in range(3)])
    v_sum = vs[0] + vs[1]  # the all-reduce
    for rank in range(world):
        lora_expand(v_sum[:, :R], yd[rank][0], seg_slot, seg_off, seg_rank, pool=pools[rank], layer=0, proj=0,
                    perm=perm)
        lora_expand_multi(v_sum[:, R:], yd[rank][1:], seg_slot, seg_off, seg_rank, pool=pools[rank], layer=0,
                          projs=[1, 2], perm=perm)
    torch.cuda.synchronize()
    for p in range(3):
        got = torch.cat([yd[r][p] for r in range(world)], dim=1).float().cpu().numpy()
        ref = lora_apply_ref(x, ys[p], perm, seg_off, seg_slot, seg_rank, full[p])
        np.testing.assert_allclose(got, ref, rtol=BF16_RTOL, atol=BF16_ATOL)
    for pool in pools:
        pool.close()


def _run_slots(dtype, h_in, h_out, slot_ranks, req_slots, req_ntok, seed, n_slots, max_tokens=4096):
    """_run_case with an explicit slot capacity (catalog-sized pools)."""
    from paper_2411_17741_b200.ops import lora_apply

    rng = np.random.default_rng(seed)
    bf16 = dtype == torch.bfloat16
    adapters = make_adapters(rng, slot_ranks, h_in, h_out, bf16=bf16)
    T = int(np.sum(req_ntok))
    x = rng.standard_normal((T, h_in)).astype(np.float32)
    y0 = rng.standard_normal((T, h_out)).astype(np.float32)
    if bf16:
        x, y0 = bf16_round(x), bf16_round(y0)
    npages = sum(-(-r // 8) for r in slot_ranks.values())
    pool = _pool(1, [h_in], [h_out], dtype, npages, n_slots=n_slots, max_tokens=max_tokens)
    _install(pool, {s: [adapters[s]] for s in slot_ranks}, slot_ranks, device_pack=True)
    req_rank = [slot_ranks[s] if s >= 0 else 0 for s in req_slots]
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(req_slots, req_rank, req_ntok)
    xd = torch.from_numpy(x).to("cuda", dtype)
    yd = torch.from_numpy(y0).to("cuda", dtype)
    lora_apply(xd, yd, seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=0, perm=perm)
    torch.cuda.synchronize()
    got = yd.float().cpu().numpy()
    ref = lora_apply_ref(x, y0, perm, seg_off, seg_slot, seg_rank, adapters)
    pool.close()
    return got, ref


def test_c2_full_batch_one_layer_proj_bf16():
    """C2 at full size for one (layer, proj): the seed-0 decode batch of 256 tokens over the
    100-adapter catalog (82 distinct adapters, ranks 8-128), Llama-2-7B h=4096, bf16."""
    from paper_2411_17741_b200.model import build_catalog
    from paper_2411_17741_b200.workload import decode_batch

    catalog = build_catalog(100)
    ids = list(catalog)
    slot_of = {a: i for i, a in enumerate(ids)}
    slot_ranks = {i: catalog[a].rank for i, a in enumerate(ids)}
    batch = decode_batch(0, 256, 100)
    assert len(set(batch)) == 82
    got, ref = _run_slots(torch.bfloat16, 4096, 4096, slot_ranks, [slot_of[a] for a in batch], [1] * 256,
                          seed=41, n_slots=100)
    np.testing.assert_allclose(got, ref, rtol=BF16_RTOL, atol=BF16_ATOL)


def test_maximum_segments_and_tokens():
    """The limits at once: 512 segments (kMaxSegments), 4096 tokens (max_tokens), ranks up to
    128 (kMaxRank); 8-token requests stay on the decode kernel, fp32 rtol 1e-5."""
    rng = np.random.default_rng(77)
    ranks = [8, 16, 32, 64, 128, 24, 40, 120]
    slot_ranks = {s: ranks[s % len(ranks)] for s in range(512)}
    req_slots = rng.permutation(512).tolist()
    got, ref = _run_slots(torch.float32, 256, 128, slot_ranks, req_slots, [8] * 512, seed=78, n_slots=512)
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-4)


def test_tensor_parallel_degree1_uses_fused_apply():
    """TensorParallelLora at TP degree 1 (no exchange step) runs the fused apply per run of
    projections sharing h_out (q alone, k+v together under GQA) and must equal the oracle."""
    from paper_2411_17741_b200.tp import TensorParallelLora

    rng = np.random.default_rng(19)
    H_IN, H_OUT = [1024, 1024, 1024], [1024, 128, 128]
    slot_ranks = {0: 64, 1: 16, 2: 8}
    full = [make_adapters(rng, slot_ranks, H_IN[p], H_OUT[p], bf16=True) for p in range(3)]
    req_slots = rng.integers(0, 3, 30).tolist()
    req_rank = [slot_ranks[s] for s in req_slots]
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(req_slots, req_rank, [1] * 30)
    x = bf16_round(rng.standard_normal((30, 1024)).astype(np.float32))
    ys = [bf16_round(rng.standard_normal((30, H_OUT[p])).astype(np.float32)) for p in range(3)]
    pool = _pool(1, H_IN, H_OUT, torch.bfloat16, 3 * 8, max_tokens=256)
    _install(pool, {s: [full[p][s] for p in range(3)] for s in slot_ranks}, slot_ranks)
    tp = TensorParallelLora(pool, max_tokens=256, r_stride=64, proj_groups=[[0, 1, 2]], group=False)
    xd = torch.from_numpy(x).to("cuda", torch.bfloat16)
    yd = [torch.from_numpy(ys[p]).to("cuda", torch.bfloat16) for p in range(3)]
    tp.apply_layer(0, [xd], yd, seg_slot, seg_off, seg_rank, perm=perm)
    torch.cuda.synchronize()
    assert tp.allreduce_count == 0
    for p in range(3):
        ref = lora_apply_ref(x, ys[p], perm, seg_off, seg_slot, seg_rank, full[p])
        np.testing.assert_allclose(yd[p].float().cpu().numpy(), ref, rtol=BF16_RTOL, atol=BF16_ATOL)
    pool.close()


def test_device_limit_error_leaves_y_and_the_next_apply_intact():
    """A segment table the host cannot see (device count) that exceeds the pool's token limit:
    the decode kernel refuses it on the device (error word set, y untouched), and the applies
    issued after it on the same stream are exact — the refused launch still re-armed the
    counter set of the apply before it, which the next apply reuses.
    Ranks 128/64 make more units than CTAs (dynamic claims), and every apply has new inputs,
    so stale counters would show up as missing or early expand work."""
    from paper_2411_17741_b200.ops import lora_apply

    rng = np.random.default_rng(11)
    h = 1024
    slot_ranks = {0: 128, 1: 64}
    adapters = make_adapters(rng, slot_ranks, h, h, bf16=True)
    pool = _pool(1, [h], [h], torch.bfloat16, 24, n_slots=2, max_tokens=64)
    pool.set_prefill_route(0)  # decode kernel only
    _install(pool, {s: [adapters[s]] for s in slot_ranks}, slot_ranks)
    pool.device_error(clear=True)
    seg_off = [0, 20, 50]

    def checked_apply():
        x0 = bf16_round(rng.standard_normal((50, h)).astype(np.float32))
        y0 = bf16_round(rng.standard_normal((50, h)).astype(np.float32))
        yd = torch.from_numpy(y0).cuda().to(torch.bfloat16)
        lora_apply(torch.from_numpy(x0).cuda().to(torch.bfloat16), yd, [0, 1], seg_off, [128, 64], pool=pool,
                   layer=0, proj=0)
        torch.cuda.synchronize()
        ref = lora_apply_ref(x0, y0, np.arange(50), np.array(seg_off), np.array([0, 1]), np.array([128, 64]),
                             adapters)
        np.testing.assert_allclose(yd.float().cpu().numpy(), bf16_round(ref.astype(np.float32)), rtol=BF16_RTOL,
                                   atol=BF16_ATOL)

    checked_apply()  # leaves its counter set dirty: the refused launch below must re-arm it
    x = torch.from_numpy(bf16_round(rng.standard_normal((50, h)).astype(np.float32))).cuda().to(torch.bfloat16)
    y = torch.from_numpy(bf16_round(rng.standard_normal((50, h)).astype(np.float32))).cuda().to(torch.bfloat16)
    y_before = y.clone()
    n_dev = torch.tensor([2], dtype=torch.int32, device="cuda")
    # 80 tokens in the (device-counted) table of a 64-token pool
    lora_apply(x, y, [0, 1], [0, 40, 80], [128, 64], pool=pool, layer=0, proj=0, n_seg_dev=n_dev)
    torch.cuda.synchronize()
    assert pool.device_error(clear=True) != 0
    assert torch.equal(y, y_before)
    for _ in range(3):  # both counter parities after the refused launch
        checked_apply()
    assert pool.device_error(clear=True) == 0
    pool.close()
