"""Regenerate tests/golden/* from the unmodified reference (test infrastructure only).

Run in the build container, where /root/reference exists:
    python oracle/gen_golden.py
The GPU box has no /root/reference; tests there read the frozen JSON fixtures.

Fixtures
  cache_traces.json   random op traces driven through the reference AdapterCache
                      (adapter_cache.py:65-328) for every policy / prefetch mode; every
                      return value, exception, counter and the resident set after each op.
  workload_draws.json assign_adapter draws (workload.py:55-64) for the C2 batches (seeds
                      0/1/2, 256 tokens) and adapter-level Zipf draws (workload.py:220-226).
  sim_batches.json    per-step (prefills, decoders) batches captured at the LoRA seam of the
                      reference simulate() (engine.py:443-447) with the reference's own
                      adapter_units for the step (engine.py:64-76).
  cost_solo.json      CostModel.prefill_step_us / decode_steps_us (engine.py:80-97) on a
                      grid of (input, output, rank) for two parameter sets.
  batch_results.json  MultiQueueScheduler.generate_batch results (scheduler.py:528-550)
                      against a scripted oracle (the reference test's hand trace plus
                      random queue layouts) and FifoScheduler cases: admitted order +
                      budget ledger.
"""
from __future__ import annotations

import json
import random
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"


def _import_ref():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import adaptersim  # noqa: F401
    from adaptersim import adapter_cache, engine, model, scheduler, workload

    return adapter_cache, engine, model, scheduler, workload


def cache_traces(n_traces: int = 24, n_ops: int = 600):
    ac, _, model, _, _ = _import_ref()
    out = []
    policies = ["cost-aware", "lru", "fairshare", "none"]
    prefetch = ["off", "queue-driven", "histogram"]
    for i in range(n_traces):
        rng = random.Random(1000 + i)
        pol = policies[i % len(policies)]
        pf = prefetch[(i // len(policies)) % len(prefetch)]
        ranks = (8, 16, 32, 64, 128)
        per_rank = 3 + i % 4
        catalog = {}
        for r in ranks:
            for j in range(per_rank):
                aid = f"r{r}-{j}"
                catalog[aid] = model.make_adapter_spec(aid, r)
        window = [2_000, 50_000, 10 ** 9][i % 3]
        cfg = model.CacheConfig(policy=model.CachePolicy(pol), frequency_window_us=window,
                                prefetch=model.PrefetchMode(pf))
        cache = ac.AdapterCache(cfg, catalog)
        ids = list(catalog)
        ops = []
        now = 0
        held: list[str] = []
        cap = rng.choice([400, 800, 1600, 3000])
        r0 = cache.set_capacity(cap, set(), now)
        ops.append({"op": "set_capacity", "args": [cap, [], now], "ret": r0})
        for _ in range(n_ops):
            now += rng.randint(0, 400)
            x = rng.random()
            rec = None
            if x < 0.30:
                aid = rng.choice(ids)
                res = cache.acquire(aid, now)
                rec = {"op": "acquire", "args": [aid, now], "ret": [res.hit, res.load_bytes]}
                if res.hit:
                    held.append(aid)
            elif x < 0.45:
                aid = rng.choice(ids)
                e = cache.lookup(aid)
                hints = sorted(rng.sample(ids, rng.randint(0, 4)))
                if not e.resident and not e.loading:
                    try:
                        ev = cache.evict_until(e.size_tokens, set(hints), now)
                        rec = {"op": "evict_until", "args": [e.size_tokens, hints, now], "ret": ev}
                    except ac.InsufficientEvictableMemory:
                        rec = {"op": "evict_until", "args": [e.size_tokens, hints, now], "raises": "InsufficientEvictableMemory"}
                    ops.append(rec)
                    if "raises" not in rec:
                        cache.begin_load(aid, now)
                        ops.append({"op": "begin_load", "args": [aid, now], "ret": None})
                    rec = None
            elif x < 0.55:
                loading = [a for a in ids if cache.lookup(a).loading]
                if loading:
                    aid = rng.choice(loading)
                    cache.finish_load(aid, now)
                    rec = {"op": "finish_load", "args": [aid, now], "ret": None}
                    if rng.random() < 0.7:
                        ops.append(rec)
                        cache.take_ref(aid, now)
                        held.append(aid)
                        rec = {"op": "take_ref", "args": [aid, now], "ret": None}
            elif x < 0.75 and held:
                aid = held.pop(rng.randrange(len(held)))
                cache.release(aid, now)
                rec = {"op": "release", "args": [aid, now], "ret": None}
            elif x < 0.85:
                cap = rng.randrange(200, 3500)
                hints = sorted(rng.sample(ids, rng.randint(0, 5)))
                ev = cache.set_capacity(cap, set(hints), now)
                rec = {"op": "set_capacity", "args": [cap, hints, now], "ret": ev}
            elif x < 0.92:
                aid = rng.choice(ids)
                cache.note_arrival(aid, now)
                rec = {"op": "note_arrival", "args": [aid, now], "ret": None}
            else:
                queued = [rng.choice(ids) for _ in range(rng.randint(0, 6))]
                free = cache.free_tokens
                ret = cache.prefetch_candidates(queued, free, now)
                rec = {"op": "prefetch_candidates", "args": [queued, free, now], "ret": ret}
            if rec is not None:
                ops.append(rec)
            # invalid op probes (CacheFault) now and then
            if rng.random() < 0.02:
                aid = rng.choice(ids)
                try:
                    cache.release(aid, now)
                    held_rm = aid in held
                    if held_rm:
                        held.remove(aid)
                    ops.append({"op": "release", "args": [aid, now], "ret": None})
                except ac.CacheFault:
                    ops.append({"op": "release", "args": [aid, now], "raises": "CacheFault"})
            ops[-1]["state"] = {
                "used": cache.used_tokens, "cap": cache.capacity_tokens, "ne": cache.non_evictable_tokens,
                "hits": cache.hits, "misses": cache.misses, "evictions": cache.evictions, "loads": cache.loads,
                # resident set as a bitmask over the catalog order
                "resident": sum(1 << k for k, a in enumerate(ids) if cache.lookup(a).resident),
            }
        # a score probe over the eligible set at the end
        elig = cache._eligible()
        scores = {e.spec.adapter_id: cache.score(e, elig, now) for e in elig}
        out.append({"policy": pol, "prefetch": pf, "window_us": window, "ranks": list(ranks), "per_rank": per_rank,
                    "ops": ops, "final_scores": scores, "final_now": now})
    return out


def workload_draws():
    _, _, model, _, wl = _import_ref()
    cfg = model.WorkloadConfig(num_adapters=100)
    hw = model.HardwareProfile()
    catalog = wl.build_catalog(cfg, hw)
    out = {"catalog_ids": list(catalog), "decode": {}, "zipf": {}}
    for seed in (0, 1, 2):
        rng = np.random.default_rng(seed)
        out["decode"][str(seed)] = [wl.assign_adapter(rng, cfg, catalog) for _ in range(256)]
    # adapter-level Zipf (write_mixed_trace convention): reproduce the id/prob tables and draws
    for seed in (0, 1):
        n, s = 1000, 0.7
        raw = [(i + 1) ** -s for i in range(n)]
        z = sum(raw)
        ids = [f"r{sorted((8, 16, 32, 64, 128))[i % 5]}-{i // 5}" for i in range(n)]
        probs = [r / z for r in raw]
        rng = np.random.default_rng(seed)
        out["zipf"][str(seed)] = [ids[int(rng.choice(n, p=probs))] for _ in range(256)]
    return out


def sim_batches(max_steps: int = 400):
    _, engine, model, _, _ = _import_ref()
    cfg = model.SimulationConfig()
    cfg.workload.arrival_rate = 6.0
    cfg.workload.duration_s = 20.0
    cfg.workload.num_adapters = 100
    cfg.workload.seed = 3
    captured = []
    orig = engine.CostModel.step_duration

    def spy(self, prefills, decoders, rank_of):
        if len(captured) < max_steps:
            units = 0
            for r in decoders:
                units += rank_of[r.spec.adapter_id]
            for r in prefills:
                units += rank_of[r.spec.adapter_id] * r.spec.input_tokens
            captured.append({
                "prefills": [[r.spec.adapter_id, r.spec.input_tokens] for r in prefills],
                "decoders": [r.spec.adapter_id for r in decoders],
                "decoder_active": [r.spec.input_tokens + r.tokens_generated for r in decoders],
                "adapter_units": units,
                "duration_us": orig(self, prefills, decoders, rank_of),
            })
        return orig(self, prefills, decoders, rank_of)

    engine.CostModel.step_duration = spy
    try:
        engine.simulate(cfg)
    finally:
        engine.CostModel.step_duration = orig
    return {"config": "SimulationConfig() with arrival_rate=6, duration_s=20, num_adapters=100, seed=3",
            "steps": captured}


def batch_results():
    """MultiQueueScheduler.generate_batch (scheduler.py:528-550, Algorithm 1: per-queue quota
    phase, then leftover in queue order) on scripted queues — the hand trace of the
    reference's own test (test_scheduler.py:222-232) plus random layouts — and FifoScheduler
    cases; each with the admitted order and the budget ledger."""
    _, _, model, sched, _ = _import_ref()
    out = []
    rng = random.Random(7)

    class Oracle:
        def __init__(self, blocked=()):
            self.blocked = set(blocked)

        def adapter_charge(self, state):
            return 0

        def adapter_fits_free(self, state):
            return True

        def try_admit(self, state, now):
            return sched.AdmitOutcome(state.request_id not in self.blocked, "adapter")

        def head_memory_eta(self, state, now):
            return now + 1000

        def estimate_completion(self, state, now):
            return now + 10

    def mlq(queue_needs, quotas, adapters):
        cfg = model.SchedulerConfig(policy=model.SchedulerPolicy.MLQ)
        s = sched.MultiQueueScheduler(cfg, sum(quotas), lambda aid: int(aid[1:].split("-")[0]), lambda r: 4 * r,
                                      lambda i, o, r: 1000, [8, 16, 32, 64, 128])
        s.layout = sched.QueueLayout(len(queue_needs), [], [0.0] * (len(queue_needs) - 1), [])
        s.queues = [[] for _ in queue_needs]
        s.quotas = list(quotas)
        s.borrowed = [0] * len(queue_needs)
        rid = 0
        for q, needs in enumerate(queue_needs):
            for need in needs:
                half = need // 2
                spec = model.RequestSpec(rid, rid, half, 1, adapters[rid % len(adapters)])
                st = model.RequestState(spec, predicted_output_tokens=need - half)
                st.queue_index = q
                s.queues[q].append(st)
                s.pending_ids.add(rid)
                rid += 1
        return s

    def record(kind, res, extra=None):
        d = {"scheduler": kind,
             "admitted": [[st.request_id, st.spec.adapter_id, st.spec.input_tokens] for st in res.admitted],
             "admitted_need": [st.borrowed_quota for st in res.admitted],
             "budgets": res.budgets, "consumed": res.consumed, "leftover": res.leftover, "stranded": res.stranded}
        d.update(extra or {})
        out.append(d)

    # the reference test's hand trace (test_scheduler.py:222-232)
    s = mlq([[30, 30, 30, 30], [40], [50, 80]], [100, 100, 100], ["r8-0"])
    record("mlq", s.generate_batch(0, Oracle()), {"case": "hand-trace"})
    ads = [f"r{r}-{j}" for r in (8, 16, 32, 64, 128) for j in range(3)]
    for case in range(16):
        nq = rng.randint(1, 4)
        needs = [[rng.randint(8, 120) for _ in range(rng.randint(0, 8))] for _ in range(nq)]
        quotas = [rng.randint(0, 300) for _ in range(nq)]
        nreq = sum(len(n) for n in needs)
        blocked = {i for i in range(nreq) if rng.random() < 0.15}
        s = mlq(needs, quotas, ads)
        record("mlq", s.generate_batch(500, Oracle(blocked)), {"case": f"random-{case}"})
    for case in range(6):
        cfg = model.SchedulerConfig()
        s = sched.FifoScheduler(cfg, 4000, lambda aid: int(aid[1:].split("-")[0]))
        for i in range(rng.randint(5, 30)):
            r = rng.choice([8, 16, 32, 64, 128])
            spec = model.RequestSpec(i, i * 10, rng.randint(16, 600), rng.randint(1, 200), f"r{r}-{rng.randint(0, 3)}")
            st = model.RequestState(spec, rng.randint(1, 200))
            s.on_arrival(st, i * 10)
        record("fifo", s.generate_batch(500, Oracle({i for i in range(40) if i % 7 == 5})), {"case": f"fifo-{case}"})
    return out


def cost_solo():
    """CostModel.prefill_step_us / decode_steps_us (engine.py:80-97) on a grid of (input tokens,
    output tokens, rank) with the default and a non-default CostModelParams."""
    _, engine, model, _, _ = _import_ref()
    out = []
    for params in (model.CostModelParams(), model.CostModelParams(prefill_base_us=1234.5, prefill_per_token_us=7.25,
                                                                 decode_base_us=987.0, decode_per_token_us=3.5,
                                                                 adapter_compute_per_rank_token_us=0.377)):
        cm = engine.CostModel(params)
        rows = []
        for i in (1, 7, 64, 256, 1000, 2048):
            for o in (0, 1, 2, 17, 300, 1024):
                for r in (8, 16, 32, 64, 128):
                    rows.append([i, o, r, cm.prefill_step_us(i, r), cm.decode_steps_us(i, o, r)])
        out.append({"params": {k: getattr(params, k) for k in ("prefill_base_us", "prefill_per_token_us",
                                                              "decode_base_us", "decode_per_token_us",
                                                              "adapter_compute_per_rank_token_us")},
                    "rows": rows})
    return out


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    (OUT / "cache_traces.json").write_text(json.dumps(cache_traces()))
    (OUT / "workload_draws.json").write_text(json.dumps(workload_draws()))
    (OUT / "sim_batches.json").write_text(json.dumps(sim_batches()))
    (OUT / "batch_results.json").write_text(json.dumps(batch_results()))
    (OUT / "cost_solo.json").write_text(json.dumps(cost_solo()))
    for f in sorted(OUT.glob("*.json")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
