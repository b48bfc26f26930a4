"""C4 replica serving loop on the CPU (fake pool; fills complete a few polls after they are
issued): the loop's recorded decision trace replays bit-exactly through a fresh AdapterCache
and — when /root/reference is present — through the UNMODIFIED reference AdapterCache
(adapter_cache.py:65-328) fed that replica's sub-trace; every request is
executed exactly once, only with its adapter resident; prefetches are issued for queued
adapters (engine.py:457-470) and completions are driven by poll_fills (engine.py:294-301)."""
import numpy as np
import pytest

import _fakes
from paper_2411_17741_b200.adapter_cache import AdapterCache
from paper_2411_17741_b200.model import CacheConfig, CachePolicy, PrefetchMode, make_adapter_spec, zipf_catalog
from paper_2411_17741_b200.serving import ReplicaLoop, replay_ops


def _run(policy="cost-aware", prefetch="queue-driven", n_adapters=200, cap_pages=180, steps=60, per_step=64,
         delay=3, seed=0):
    ids, probs = zipf_catalog(n_adapters)
    catalog = {a: make_adapter_spec(a, int(a[1:].split("-")[0])) for a in ids}
    cfg = CacheConfig(policy=CachePolicy(policy), prefetch=PrefetchMode(prefetch))
    _fakes.Event.delay = delay
    try:
        cache, log = _fakes.paged_cache(cfg, catalog, cap_pages)
        batches = []

        def run_batch(slots, ranks, ntok):
            for s in slots:
                aid = ids[int(s)]
                assert cache.lookup(aid).resident and cache.lookup(aid).rc > 0, aid
            batches.append(list(map(int, slots)))

        loop = ReplicaLoop(cache, catalog, run_batch, capacity_tokens=cap_pages * 32,
                           prefetch=prefetch != "off", max_admit=per_step)
        rng = np.random.default_rng(seed)
        arrived = 0
        for _ in range(steps):
            n = int(rng.integers(0, 2 * per_step))  # bursts beyond the per-step admission budget
            arr = [ids[int(k)] for k in rng.choice(len(ids), n, p=np.asarray(probs))]
            arrived += len(arr)
            loop.step(arr)
        for _ in range(delay + 40):  # drain the queue and the in-flight fills
            loop.step([])
    finally:
        _fakes.Event.delay = 0
    return cfg, catalog, cache, loop, batches, arrived


@pytest.mark.parametrize("policy,prefetch", [("cost-aware", "queue-driven"), ("lru", "off"),
                                             ("fairshare", "histogram"), ("cost-aware", "off")])
def test_replica_decisions_replay_through_fresh_cache(policy, prefetch):
    cfg, catalog, cache, loop, batches, arrived = _run(policy, prefetch)
    ops = cache.op_log
    assert len(ops) > 1000
    fresh = AdapterCache(cfg, catalog)
    assert replay_ops(fresh, ops) == []
    for k in ("hits", "misses", "evictions", "loads", "used_tokens", "capacity_tokens"):
        assert getattr(fresh, k) == getattr(cache, k), k
    # conservation: every arrival was executed once, or is still deferred / waiting
    waiting = sum(loop.waiters.values())
    assert loop.stats["executed"] + len(loop.deferred) + waiting == arrived
    assert sum(len(b) for b in batches) == loop.stats["executed"]
    assert cache.evictions > 0 and cache.misses > 0 and loop.stats["completed"] > 0
    if prefetch != "off":
        assert loop.stats["prefetches"] > 0


@pytest.mark.reference
@pytest.mark.parametrize("policy,prefetch", [("cost-aware", "queue-driven"), ("lru", "histogram"),
                                             ("none", "off")])
def test_replica_decisions_bit_exact_vs_reference_cache(reference_pkg, policy, prefetch):
    from adaptersim import adapter_cache as ref_ac
    from adaptersim import model as ref_model

    cfg, catalog, cache, loop, batches, arrived = _run(policy, prefetch, seed=1)
    ref_cfg = ref_model.CacheConfig(policy=ref_model.CachePolicy(policy), prefetch=ref_model.PrefetchMode(prefetch))
    ref_cat = {a: ref_model.make_adapter_spec(a, s.rank) for a, s in catalog.items()}
    ref = ref_ac.AdapterCache(ref_cfg, ref_cat)
    assert replay_ops(ref, cache.op_log) == []
    assert (ref.hits, ref.misses, ref.evictions, ref.loads, ref.used_tokens) == (
        cache.hits, cache.misses, cache.evictions, cache.loads, cache.used_tokens)
    resident = sorted(a for a, e in ref.entries.items() if e.resident)
    assert resident == sorted(a for a, e in cache.entries.items() if e.resident)


def test_replay_detects_a_divergent_decision():
    cfg, catalog, cache, loop, batches, arrived = _run(steps=20)
    ops = [dict(r) for r in cache.op_log]
    i = next(k for k, r in enumerate(ops) if r["op"] == "acquire" and r["ret"][0])
    ops[i] = dict(ops[i], ret=[False, ops[i]["ret"][1]])
    assert replay_ops(AdapterCache(cfg, catalog), ops)
