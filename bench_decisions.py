"""CPU decision-path timings for bench.py (SURVEY §8d "CPU path").

The reference's own Python decision path, imported UNMODIFIED from `baseline/_ref` (the
offline install of /root/reference, which travels to the GPU box), timed on one host core:

  * AdapterCache (adapter_cache.py:65-328) at 1000 adapters (Zipf 0.7 catalog, the
    write_mixed_trace convention, workload.py:220-226) with capacity = 10% of the catalog's
    tokens: a Zipf request stream through acquire / evict_until / begin_load / finish_load /
    take_ref / release — requests/s and ms per eviction;
  * the same stream through this repo's AdapterCache (O(E) scoring, O(1) pinned counter),
    with every decision compared (hits, misses, evicted ids in order);
  * simulate() (engine.py:585-592) wall time on a 1000-adapter config, with the number of
    MultiQueueScheduler.generate_batch calls (scheduler.py:528-550) and their rate.

Returns a dict for the bench line; {"unavailable": why} when baseline/_ref is absent.
"""
from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
REF = ROOT / "baseline" / "_ref"


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def _import_ref():
    if not (REF / "adaptersim").exists():
        return None
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import adaptersim  # noqa: F401
    from adaptersim import adapter_cache, engine, model, scheduler

    return adapter_cache, engine, model, scheduler


def _zipf_stream(n_adapters: int, n_req: int, seed: int, s: float = 0.7):
    ids = [f"r{sorted((8, 16, 32, 64, 128))[i % 5]}-{i // 5}" for i in range(n_adapters)]
    raw = np.array([(i + 1) ** -s for i in range(n_adapters)])
    p = raw / raw.sum()
    rng = np.random.default_rng(seed)
    return ids, [ids[int(k)] for k in rng.choice(n_adapters, n_req, p=p)]


def _drive(cache, stream, exc_type):
    """One request per 1 ms of reference time: acquire; on a miss evict_until + begin_load +
    finish_load + take_ref; then release.  Returns the decision log and counters."""
    log = []
    evictions = 0
    now = 0
    for aid in stream:
        now += 1000
        r = cache.acquire(aid, now)
        if r.hit:
            log.append(("h", aid))
        else:
            e = cache.lookup(aid)
            try:
                ev = cache.evict_until(e.spec.size_tokens, {aid}, now)
            except exc_type:
                log.append(("d", aid))
                continue
            evictions += len(ev)
            log.append(("m", aid, tuple(ev)))
            cache.begin_load(aid, now)
            cache.finish_load(aid, now)
            cache.take_ref(aid, now)
        cache.release(aid, now)
    return log, evictions


def decision_path(n_req: int = 3000, sim_duration_s: float = 600.0) -> dict:
    ref = _import_ref()
    if ref is None:
        return {"unavailable": "baseline/_ref (offline install of the reference) is not present"}
    r_ac, r_engine, r_model, r_sched = ref
    from paper_2411_17741_b200.adapter_cache import AdapterCache, InsufficientEvictableMemory
    from paper_2411_17741_b200.model import CacheConfig, make_adapter_spec

    ids, stream = _zipf_stream(1000, n_req, seed=0)
    ref_catalog = {a: r_model.make_adapter_spec(a, int(a[1:].split("-")[0])) for a in ids}
    our_catalog = {a: make_adapter_spec(a, int(a[1:].split("-")[0])) for a in ids}
    cap = sum(s.size_tokens for s in ref_catalog.values()) // 10

    rc = r_ac.AdapterCache(r_model.CacheConfig(), ref_catalog)
    rc.set_capacity(cap, set(), 0)
    t0 = time.perf_counter()
    ref_log, ref_ev = _drive(rc, stream, r_ac.InsufficientEvictableMemory)
    t_ref = time.perf_counter() - t0

    oc = AdapterCache(CacheConfig(), our_catalog)
    oc.set_capacity(cap, set(), 0)
    t0 = time.perf_counter()
    our_log, our_ev = _drive(oc, stream, InsufficientEvictableMemory)
    t_our = time.perf_counter() - t0

    # simulate(): the reference engine end to end, generate_batch calls counted and timed
    cfg = r_model.SimulationConfig()
    cfg.workload.num_adapters = 1000
    cfg.workload.duration_s = sim_duration_s
    cls = r_sched.MultiQueueScheduler
    orig = cls.generate_batch
    stats = {"n": 0, "t": 0.0}

    def timed(self, now, oracle):
        t = time.perf_counter()
        try:
            return orig(self, now, oracle)
        finally:
            stats["n"] += 1
            stats["t"] += time.perf_counter() - t

    cls.generate_batch = timed
    try:
        t0 = time.perf_counter()
        res = r_engine.simulate(cfg)
        t_sim = time.perf_counter() - t0
    finally:
        cls.generate_batch = orig
    n_done = len(getattr(res, "records", []) or [])
    return {
        "kind": "reference (unmodified adaptersim from baseline/_ref), one host core",
        "cpu_model": cpu_model(),
        "cores": 1,
        "adapter_cache": {
            "catalog": "1000 adapters, Zipf 0.7 (write_mixed_trace ids), capacity 10% of catalog tokens",
            "requests": n_req,
            "reference_requests_per_s": n_req / t_ref,
            "reference_ms_per_eviction": t_ref * 1e3 / max(1, ref_ev),
            "ours_requests_per_s": n_req / t_our,
            "ours_ms_per_eviction": t_our * 1e3 / max(1, our_ev),
            "evictions": ref_ev,
            "hit_rate": sum(1 for x in ref_log if x[0] == "h") / n_req,
            "decisions_identical": ref_log == our_log,
        },
        "simulate": {
            "config": f"SimulationConfig(), num_adapters=1000, duration_s={sim_duration_s:g}",
            "wall_s": t_sim,
            "requests": n_done,
            "generate_batch_calls": stats["n"],
            "generate_batch_calls_per_s": stats["n"] / stats["t"] if stats["t"] > 0 else None,
            "generate_batch_share_of_wall": stats["t"] / t_sim if t_sim > 0 else None,
        },
    }


if __name__ == "__main__":
    import json

    sys.path.insert(0, str(ROOT))
    print(json.dumps(decision_path(), indent=1))
