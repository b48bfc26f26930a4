"""AdapterCache decisions: bit-exact with the reference (adapter_cache.py:65-328).

1. Replays of frozen reference traces (tests/golden/cache_traces.json, made by
   oracle/gen_golden.py from the unmodified reference) through our AdapterCache: every
   return value, exception, counter and resident set must match.
2. The reference test suite's known answers (test_cache.py:63-355), restated.
3. When /root/reference is present: live differential traces against the reference.
"""
import json
import math
import random
from collections import deque

import pytest

from paper_2411_17741_b200.adapter_cache import (AdapterCache, AdapterEntry, CacheFault,
                                                 InsufficientEvictableMemory)
from paper_2411_17741_b200.model import (CacheConfig, CachePolicy, PrefetchMode, US_PER_SEC,
                                         build_catalog, make_adapter_spec)


def _catalog(ranks, per_rank):
    cat = {}
    for r in ranks:
        for j in range(per_rank):
            aid = f"r{r}-{j}"
            cat[aid] = make_adapter_spec(aid, r)
    return cat


def _replay(trace):
    cat = _catalog(trace["ranks"], trace["per_rank"])
    ids = list(cat)
    cfg = CacheConfig(policy=CachePolicy(trace["policy"]), frequency_window_us=trace["window_us"],
                      prefetch=PrefetchMode(trace["prefetch"]))
    cache = AdapterCache(cfg, cat)
    for i, rec in enumerate(trace["ops"]):
        op, args = rec["op"], rec["args"]
        where = f"op {i} {op}{tuple(args)}"
        if op == "acquire":
            r = cache.acquire(*args)
            assert [r.hit, r.load_bytes] == rec["ret"], where
        elif op == "evict_until":
            if "raises" in rec:
                with pytest.raises(InsufficientEvictableMemory):
                    cache.evict_until(args[0], set(args[1]), args[2])
            else:
                assert cache.evict_until(args[0], set(args[1]), args[2]) == rec["ret"], where
        elif op == "set_capacity":
            assert cache.set_capacity(args[0], set(args[1]), args[2]) == rec["ret"], where
        elif op == "begin_load":
            cache.begin_load(*args)
        elif op == "finish_load":
            cache.finish_load(*args)
        elif op == "take_ref":
            cache.take_ref(*args)
        elif op == "release":
            if "raises" in rec:
                with pytest.raises(CacheFault):
                    cache.release(*args)
            else:
                cache.release(*args)
        elif op == "note_arrival":
            cache.note_arrival(*args)
        elif op == "prefetch_candidates":
            assert cache.prefetch_candidates(args[0], args[1], args[2]) == rec["ret"], where
        else:  # pragma: no cover
            raise AssertionError(op)
        st = rec.get("state")
        if st is not None:
            got = {"used": cache.used_tokens, "cap": cache.capacity_tokens, "ne": cache.non_evictable_tokens,
                   "hits": cache.hits, "misses": cache.misses, "evictions": cache.evictions, "loads": cache.loads,
                   "resident": sum(1 << k for k, a in enumerate(ids) if cache.lookup(a).resident)}
            assert got == st, where
            assert cache.non_evictable_tokens == cache.non_evictable_tokens_recount(), where
            assert cache.used_tokens == cache.resident_tokens_recount(), where
    elig = cache._eligible()
    now = trace["final_now"]
    got_scores = {e.spec.adapter_id: cache.score(e, elig, now) for e in elig}
    assert got_scores == trace["final_scores"]  # float64, bit-exact


def _traces(golden_dir):
    return json.loads((golden_dir / "cache_traces.json").read_text())


def test_reference_traces_replay_bit_exact(golden_dir):
    traces = _traces(golden_dir)
    assert len(traces) >= 20
    for t in traces:
        _replay(t)


def test_traces_cover_every_policy_and_prefetch_mode(golden_dir):
    traces = _traces(golden_dir)
    assert {t["policy"] for t in traces} == {"cost-aware", "lru", "fairshare", "none"}
    assert {t["prefetch"] for t in traces} == {"off", "queue-driven", "histogram"}
    ops = {r["op"] for t in traces for r in t["ops"]}
    assert {"acquire", "evict_until", "set_capacity", "begin_load", "finish_load", "take_ref", "release",
            "note_arrival", "prefetch_candidates"} <= ops
    assert any("raises" in r for t in traces for r in t["ops"])


# -- known answers of the reference test-suite (restated) ---------------------------------

def _entry(rank, events, last_used):
    e = AdapterEntry(make_adapter_spec(f"r{rank}-x", rank), last_used=last_used, resident=True)
    e.use_events = deque(events)
    return e


def _cache(policy=CachePolicy.COST_AWARE, capacity=10_000, catalog=None, **kw):
    c = AdapterCache(CacheConfig(policy=policy, **kw), catalog or _catalog((8, 16, 32, 64, 128), 2))
    c.set_capacity(capacity, set(), 0)
    return c


def test_score_fixture_0_4375():
    c = _cache()
    lo, mid, hi = _entry(8, [], 10), _entry(16, [900, 950], 1000), _entry(128, [800, 850, 900, 950], 500)
    s = c.score(mid, [lo, mid, hi], now=1000)
    assert s == pytest.approx(0.45 * 0.5 + 0.10 * 1.0 + 0.45 * 0.25)
    assert s == pytest.approx(0.4375)


def test_score_bounds_and_all_equal():
    c = _cache()
    best, worst = _entry(128, [910, 920, 930, 940], 1000), _entry(8, [], 10)
    assert c.score(best, [worst, best], now=1000) == pytest.approx(1.0)
    assert c.score(worst, [worst, best], now=1000) == pytest.approx(0.0)
    a, b = _entry(32, [], 100), _entry(32, [], 100)
    assert c.score(a, [a, b], now=200) == pytest.approx(1.0)


def test_acquire_miss_reports_bytes():
    assert _cache().acquire("r32-0", 5).load_bytes == 67_108_864


def test_rc_lifecycle_and_faults():
    c = _cache()
    c.begin_load("r8-0", 0)
    with pytest.raises(CacheFault):
        c.begin_load("r8-0", 0)
    c.finish_load("r8-0", 0)
    assert c.acquire("r8-0", 5).hit and c.lookup("r8-0").rc == 1
    c.acquire("r8-0", 6)
    assert c.lookup("r8-0").frequency(10, US_PER_SEC) == 2
    c.release("r8-0", 7)
    c.release("r8-0", 8)
    assert c.lookup("r8-0").resident  # RC 0 keeps the entry
    with pytest.raises(CacheFault):
        c.release("r8-0", 9)
    with pytest.raises(CacheFault):
        c.take_ref("r16-0", 9)
    with pytest.raises(CacheFault):
        c.finish_load("r16-0", 9)


def test_none_policy_drops_at_rc_zero():
    c = _cache(policy=CachePolicy.NONE)
    c.begin_load("r8-0", 0)
    c.finish_load("r8-0", 0)
    c.take_ref("r8-0", 1)
    c.release("r8-0", 2)
    assert not c.lookup("r8-0").resident and c.used_tokens == 0


def test_evict_until_atomic_and_never_rc_positive():
    cat = _catalog((8, 16), 2)
    c = _cache(capacity=96, catalog=cat)
    for a in ("r8-0", "r16-0"):
        c.begin_load(a, 0)
        c.finish_load(a, 0)
    c.acquire("r16-0", 1)  # pinned
    with pytest.raises(InsufficientEvictableMemory):
        c.evict_until(96, set(), 2)
    assert c.lookup("r8-0").resident and c.evictions == 0
    with pytest.raises(InsufficientEvictableMemory):
        c.evict_until(64, set(), 2)  # only r8-0's 32 tokens are freeable
    assert c.evict_until(32, set(), 2) == ["r8-0"]
    assert c.lookup("r16-0").resident


def test_hinted_adapters_form_second_tier():
    cat = _catalog((8,), 3)
    c = _cache(capacity=96, catalog=cat)
    for i, a in enumerate(cat):
        c.begin_load(a, i)
        c.finish_load(a, i)
    # r8-0 is the LRU victim unless hinted
    assert c.evict_until(32, {"r8-0"}, 10) == ["r8-1"]
    assert c.evict_until(64, {"r8-0"}, 11) == ["r8-2"]  # the hinted one goes last


def test_lru_matches_plain_lru_oracle():
    """LRU policy vs an independent OrderedDict LRU over 20 seeds (reference test_cache.py:283-321)."""
    from collections import OrderedDict

    for seed in range(20):
        rng = random.Random(seed)
        cat = _catalog((8, 16, 32), 4)
        c = AdapterCache(CacheConfig(policy=CachePolicy.LRU, frequency_window_us=10 ** 12), cat)
        c.set_capacity(512, set(), 0)
        lru, used, ours, theirs = OrderedDict(), 0, [], []
        now = 0
        for _ in range(300):
            now += 1
            aid = rng.choice(list(cat))
            size = cat[aid].size_tokens
            if aid in lru:
                lru.move_to_end(aid)
            else:
                while used + size > 512 and lru:
                    old, sz = lru.popitem(last=False)
                    used -= sz
                    theirs.append(old)
                lru[aid] = size
                used += size
            r = c.acquire(aid, now)
            if r.hit:
                c.release(aid, now)
            else:
                ours.extend(c.evict_until(size, set(), now))
                c.begin_load(aid, now)
                c.finish_load(aid, now)
                c.take_ref(aid, now)
                c.release(aid, now)
        assert ours == theirs, seed


def test_prefetch_queue_order_and_budget():
    c = _cache(prefetch=PrefetchMode.QUEUE_DRIVEN, capacity=400)
    # greedy in queue order: 256 + 32, r128 (512) does not fit, r16 (64) does
    got = c.prefetch_candidates(["r64-0", "r8-0", "r64-0", "r128-0", "r16-1"], 352, 5)
    assert got == ["r64-0", "r8-0", "r16-1"]
    assert c.prefetch_candidates(["r64-0", "r8-0", "r16-1"], 300, 5) == ["r64-0", "r8-0"]
    assert _cache(prefetch=PrefetchMode.OFF).prefetch_candidates(["r8-0"], 1000, 1) == []


def test_build_catalog_ids_and_byte_model():
    cat = build_catalog(100)
    assert len(cat) == 100 and list(cat)[:2] == ["r8-0", "r8-1"] and list(cat)[-1] == "r128-19"
    assert cat["r128-0"].size_bytes == 128 * 2_097_152 and cat["r128-0"].size_tokens == 512
    assert cat["r8-0"].size_tokens == 32


def test_large_catalog_eviction_is_linear_time():
    """1000 adapters with capacity at 10% of the catalog: O(E) scoring keeps an eviction
    in the tens of microseconds (the reference's O(E^2) path costs ~1.3 ms)."""
    import time

    cat = build_catalog(1000)
    c = AdapterCache(CacheConfig(), cat)
    cap = int(0.1 * sum(s.size_tokens for s in cat.values()))
    c.set_capacity(cap, set(), 0)
    rng = random.Random(0)
    ids = list(cat)
    now, n_ev, t = 0, 0, 0.0
    for _ in range(3000):
        now += 100
        aid = rng.choice(ids)
        if c.acquire(aid, now).hit:
            c.release(aid, now)
            continue
        t0 = time.perf_counter()
        ev = c.evict_until(cat[aid].size_tokens, set(), now)
        t += time.perf_counter() - t0
        n_ev += len(ev)
        c.begin_load(aid, now)
        c.finish_load(aid, now)
    assert n_ev > 100
    assert t / n_ev < 1e-3


@pytest.mark.reference
def test_live_differential_against_reference(reference_pkg):
    """Random traces through the reference AdapterCache and ours, op by op."""
    from adaptersim import adapter_cache as rac
    from adaptersim import model as rmodel

    for seed in range(6):
        rng = random.Random(seed)
        cat_r = {f"r{r}-{j}": rmodel.make_adapter_spec(f"r{r}-{j}", r) for r in (8, 16, 32, 64, 128) for j in range(6)}
        cat_o = {k: make_adapter_spec(k, v.rank) for k, v in cat_r.items()}
        pol = ["cost-aware", "lru", "fairshare"][seed % 3]
        ref = rac.AdapterCache(rmodel.CacheConfig(policy=rmodel.CachePolicy(pol), frequency_window_us=30_000), cat_r)
        ours = AdapterCache(CacheConfig(policy=CachePolicy(pol), frequency_window_us=30_000), cat_o)
        for c in (ref, ours):
            c.set_capacity(1500, set(), 0)
        ids = list(cat_r)
        now = 0
        for _ in range(1500):
            now += rng.randint(0, 300)
            aid = rng.choice(ids)
            a, b = ref.acquire(aid, now), ours.acquire(aid, now)
            assert (a.hit, a.load_bytes) == (b.hit, b.load_bytes)
            if a.hit:
                if rng.random() < 0.8:
                    ref.release(aid, now)
                    ours.release(aid, now)
                continue
            e = ref.lookup(aid)
            if e.loading:
                continue
            hints = set(rng.sample(ids, 3))
            try:
                ev_r = ref.evict_until(e.size_tokens, hints, now)
            except rac.InsufficientEvictableMemory:
                with pytest.raises(InsufficientEvictableMemory):
                    ours.evict_until(e.size_tokens, hints, now)
                continue
            assert ours.evict_until(e.size_tokens, hints, now) == ev_r
            for c in (ref, ours):
                c.begin_load(aid, now)
                c.finish_load(aid, now)
            assert ref.non_evictable_tokens == ours.non_evictable_tokens
        assert (ref.hits, ref.misses, ref.evictions, ref.loads) == (ours.hits, ours.misses, ours.evictions, ours.loads)
