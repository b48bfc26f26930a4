"""GPU: the C4 replica serving loop over the real device path — PagedAdapterCache with pinned
fills on the side stream, completions driven by poll_fills (engine.py:294-301), misses and
queue-driven prefetches issuing real copies (engine.py:491-532, 457-470), evictions reusing
pages, and every step's batch executed by LoraStepExecutor after its fills.  Every step's y
is checked against the numpy oracle with the adapters the requests name; the replica's
decision trace replays bit-exactly through a fresh AdapterCache."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle.lora_ref import bf16_round, lora_apply_ref
from oracle.segments_ref import build_segments_ref

pytestmark = pytest.mark.gpu


def _setup(n_adapters=40, cap_pages=24, h=512, n_layers=2, prefetch="queue-driven", seed=0):
    from paper_2411_17741_b200.adapter_cache import PagedAdapterCache
    from paper_2411_17741_b200.executor import LoraStepExecutor
    from paper_2411_17741_b200.model import CacheConfig, PrefetchMode, make_adapter_spec, zipf_catalog
    from paper_2411_17741_b200.pool import AdapterPool

    ids, probs = zipf_catalog(n_adapters)
    catalog = {a: make_adapter_spec(a, int(a[1:].split("-")[0])) for a in ids}
    pool = AdapterPool(cap_pages, n_layers, [h], [h], dtype=torch.bfloat16, n_slots=n_adapters, max_tokens=512)
    rng = np.random.default_rng(seed)
    weights, store = {}, {}
    for a in ids:
        r = catalog[a].rank
        al = [bf16_round((rng.standard_normal((h, r)) / np.sqrt(h)).astype(np.float32)) for _ in range(n_layers)]
        bl = [bf16_round((rng.standard_normal((r, h)) / np.sqrt(r)).astype(np.float32)) for _ in range(n_layers)]
        weights[a] = (al, bl)
        store[a] = pool.pack_host([torch.from_numpy(x) for x in al], [torch.from_numpy(x) for x in bl], r)
    s = torch.cuda.Stream()
    cache = PagedAdapterCache(CacheConfig(prefetch=PrefetchMode(prefetch)), catalog, pool, host_store=store,
                              compute_stream=s)
    ex = LoraStepExecutor(pool, max_requests=256, max_tokens=256)
    return ids, probs, catalog, pool, weights, cache, ex, s


def test_replica_loop_real_fills_outputs_and_decisions():
    from paper_2411_17741_b200.adapter_cache import AdapterCache
    from paper_2411_17741_b200.serving import ReplicaLoop, replay_ops

    ids, probs, catalog, pool, weights, cache, ex, s = _setup()
    h, L = pool.h_in[0], pool.n_layers
    rng = np.random.default_rng(1)
    checked = {"steps": 0}

    def run_batch(slots, ranks, ntok):
        T = int(ntok.sum())
        x = [bf16_round(rng.standard_normal((T, h)).astype(np.float32)) for _ in range(L)]
        y0 = [bf16_round(rng.standard_normal((T, h)).astype(np.float32)) for _ in range(L)]
        with torch.cuda.stream(s):
            xs = [[torch.from_numpy(v).to("cuda", non_blocking=False).to(torch.bfloat16)] for v in x]
            ys = [[torch.from_numpy(v).to("cuda").to(torch.bfloat16)] for v in y0]
            ex.upload(slots, ranks, ntok, stream=s)
            ex.run(xs, ys)
        s.synchronize()
        perm, off, sl, rk = build_segments_ref(slots, ranks, ntok)
        by_slot = {int(sv): ids[int(sv)] for sv in slots}
        for layer in range(L):
            ad = {sv: (weights[a][0][layer], weights[a][1][layer]) for sv, a in by_slot.items()}
            want = lora_apply_ref(x[layer], y0[layer], perm, off, sl, rk, ad)
            got = ys[layer][0].float().cpu().numpy()
            np.testing.assert_allclose(got, bf16_round(want.astype(np.float32)), rtol=2e-2, atol=2e-2)
        checked["steps"] += 1

    from paper_2411_17741_b200.adapter_cache import PagedAdapterCache

    loop = ReplicaLoop(cache, catalog, run_batch, capacity_tokens=pool.n_pages * PagedAdapterCache.TOKENS_PER_PAGE,
                       max_admit=24)
    p = np.asarray(probs)
    for i in range(40):
        n = int(rng.integers(0, 40))
        loop.step([ids[int(k)] for k in rng.choice(len(ids), n, p=p)])
    for _ in range(200):  # drain: completions arrive by event query, the host never blocks on a fill
        if not loop.deferred and not loop.in_flight:
            break
        loop.step([])
        torch.cuda.synchronize()
    pool.check_device_error()
    assert checked["steps"] > 20
    assert cache.evictions > 0 and cache.fill_count > 10 and loop.stats["completed"] > 0
    assert loop.stats["prefetches"] > 0
    assert replay_ops(AdapterCache(cache.cfg, catalog), cache.op_log) == []
    pool.close()


def test_poll_fills_reports_completed_copies_only():
    """poll_fills is an event query: an adapter appears once its pinned copy completed, and the
    step that reads it is ordered after the fill on the device (wait_ready)."""
    ids, probs, catalog, pool, weights, cache, ex, s = _setup(prefetch="off")
    cache.set_capacity(pool.n_pages * 32, set(), 0)
    a = next(x for x in ids if catalog[x].rank == 128)  # 16 pages: the largest copy
    cache.acquire(a, 1)
    cache.evict_until(catalog[a].size_tokens, set(), 1)
    cache.begin_load(a, 1)
    ev = cache.fill_event(a)
    assert ev is not None
    ev.synchronize()
    assert cache.poll_fills() == [a]
    cache.finish_load(a, 2)
    assert cache.poll_fills() == []  # no longer loading
    pool.close()
