"""Engine seams: the device path plugged into the reference's serving engine.

The reference engine (`adaptersim.engine.Simulation`) drives the adapter cache and models
the LoRA work; this module is the plugin that makes those seams real on one replica
without changing a single engine decision:

  seam (reference)                                   device work (this build)
  -------------------------------------------------  --------------------------------------------
  `Simulation.cache` (engine.py:160)                 `PagedAdapterCache`: same decisions, pages
  `_Oracle.try_admit` miss branch (engine.py:522-531) `begin_load` -> page allocation + pinned
     and `_issue_prefetches` (engine.py:457-470)        cudaMemcpyAsync on the fill stream + event
  `_on_transfer_complete` (engine.py:294-301)        the fill's completion (`poll_fills`) gates
                                                        `finish_load` / `take_ref`
  `CostModel.step_duration` (engine.py:59-78)        `LoraStepExecutor` runs the step's
     called from `_try_schedule` (engine.py:443-455)    (prefills, decoders) batch on the device

`EngineSeams.install(sim)` patches one `Simulation` instance (duck-typed: `.cache`,
`.catalog`, `.cost.step_duration`, `._on_transfer_complete`); the event loop, scheduler and
metrics stay the reference's, so `sim.run()` returns the same `RunResult` as the
unpatched engine (tests/test_serving.py) while every miss and prefetch moves real bytes and
every step executes its LoRA apply.

Fill completion modes (`fill_wait`):
  "poll"   — at the simulated completion the host waits until `poll_fills()` reports the
             adapter (the real copy gates the engine's transfer-complete event);
  "stream" — no host wait: the step that first reads the adapter orders itself after the
             fill on the device (`wait_ready`), so fills overlap the preceding steps.
Either way the step wrapper makes the compute stream wait on the fill events of every
adapter in the batch before the apply reads its pages.
"""
from __future__ import annotations

import contextlib
import time
from typing import Callable, Optional

import numpy as np

from .executor import batch_arrays


def order_after_fills(cache, adapter_ids, memo: dict) -> None:
    """Make the compute stream wait on the latest fill event of each adapter, once per event
    (`memo` remembers the event already waited on; a reload records a new one)."""
    fresh = []
    for aid in set(adapter_ids):
        ev = cache.fill_event(aid)
        if ev is not None and memo.get(aid) is not ev:
            memo[aid] = ev
            fresh.append(aid)
    if fresh:
        cache.wait_ready(sorted(fresh))


class SeamError(AssertionError):
    """The engine asked the device path for something the cache does not hold."""


class EngineSeams:
    """Device side of one replica's engine.

    cache:       a fresh `PagedAdapterCache` over the engine's catalog and cache config.
    executor:    a `LoraStepExecutor` over the cache's pool (None: decisions and fills only).
    activations: `activations(n_tokens) -> (xs_per_layer, ys_per_layer)` device buffers of the
                 step's hidden states (default: executor-sized scratch, allocated once).
    on_step:     optional `on_step(index, (slots, ranks, ntok), xs, ys)` after each chunk is
                 enqueued (tests check y against the oracle here).
    cost:        optional replacement `step_duration(prefills, decoders, rank_of)` (e.g. the
                 measured `cost_model.B200CostModel`); default keeps the engine's own.
    """

    def __init__(self, cache, executor=None, activations: Optional[Callable] = None,
                 on_step: Optional[Callable] = None, fill_wait: str = "stream", cost=None,
                 poll_timeout_s: float = 30.0):
        if fill_wait not in ("poll", "stream"):
            raise ValueError("fill_wait must be 'poll' or 'stream'")
        self.cache = cache
        self.executor = executor
        self.activations = activations
        self.on_step = on_step
        self.fill_wait = fill_wait
        self.cost = cost
        self.poll_timeout_s = float(poll_timeout_s)
        self._scratch = None
        self._ordered = {}
        # counters (reported by the C4 bench and checked by the tests)
        self.steps = 0
        self.chunks = 0
        self.tokens = 0
        self.transfers_completed = 0
        self.poll_waits = 0
        self.poll_wait_s = 0.0

    # -- install ---------------------------------------------------------------------------
    def install(self, sim) -> "EngineSeams":
        """Patch a freshly built, not yet run `Simulation` so its seams run on the device."""
        if set(sim.catalog) != set(self.cache.entries):
            raise SeamError("the cache's catalog differs from the engine's")
        if getattr(sim, "steps", 0) or getattr(sim, "arrivals_seen", 0):
            raise SeamError("install before the simulation runs")
        sim.cache = self.cache
        orig_transfer = sim._on_transfer_complete
        orig_duration = sim.cost.step_duration
        cost = self.cost

        def on_transfer_complete(adapter_id):  # engine.py:294-301
            self.transfer_complete(adapter_id)
            orig_transfer(adapter_id)

        def step_duration(prefills, decoders, rank_of):  # engine.py:59-78, called at 447
            self.run_step(prefills, decoders, rank_of)
            return (cost or orig_duration)(prefills, decoders, rank_of)

        sim._on_transfer_complete = on_transfer_complete
        sim.cost.step_duration = step_duration
        self.sim = sim
        return self

    # -- seams -----------------------------------------------------------------------------
    def transfer_complete(self, adapter_id: str) -> None:
        """The engine's transfer-complete event for `adapter_id` (before its finish_load)."""
        c = self.cache
        e = c.entries[adapter_id]
        if not e.loading:
            raise SeamError(f"transfer complete for {adapter_id}, which is not loading")
        if self.fill_wait == "poll":
            t0 = time.perf_counter()
            waited = False
            while adapter_id not in c.poll_fills():
                waited = True
                if time.perf_counter() - t0 > self.poll_timeout_s:
                    raise SeamError(f"fill of {adapter_id} did not complete in {self.poll_timeout_s} s")
                time.sleep(0)
            if waited:
                self.poll_waits += 1
                self.poll_wait_s += time.perf_counter() - t0
        self.transfers_completed += 1

    def run_step(self, prefills, decoders, rank_of) -> None:
        """Execute one engine step's LoRA work: (prefills, decoders) -> request arrays ->
        upload -> K4 + plan + every (layer, group) apply, in chunks of at most the executor's
        token capacity (requests are independent, so chunking changes nothing)."""
        self.steps += 1
        c = self.cache
        ids = [r.spec.adapter_id for r in prefills] + [r.spec.adapter_id for r in decoders]
        for aid in set(ids):
            if not c.entries[aid].resident:
                raise SeamError(f"step reads {aid}, which is not resident")
        if self.executor is None:
            return
        # the apply reads the pages after their fills
        order_after_fills(c, ids, self._ordered)
        slots, ranks, ntok = batch_arrays((prefills, decoders), c.slot_of, rank_of.__getitem__)
        cap = self.executor.max_tokens
        lo = 0
        n = len(slots)
        while lo < n:
            hi, tot = lo, 0
            while hi < n and tot + int(ntok[hi]) <= cap:
                tot += int(ntok[hi])
                hi += 1
            if hi == lo:
                raise SeamError(f"request of {int(ntok[lo])} tokens exceeds the executor's {cap}")
            self._run_chunk(slots[lo:hi], ranks[lo:hi], ntok[lo:hi])
            lo = hi

    def _run_chunk(self, slots, ranks, ntok) -> None:
        ex = self.executor
        T = int(np.sum(ntok))
        s = self.cache.compute_stream
        if self.activations is not None:
            xs, ys = self.activations(T)
        else:
            xs, ys = self._default_activations(T)
        ex.upload(slots, ranks, ntok, stream=s)
        import torch

        with (torch.cuda.stream(s) if isinstance(s, torch.cuda.Stream) else contextlib.nullcontext()):
            ex.run(xs, ys)
        self.chunks += 1
        self.tokens += T
        if self.on_step is not None:
            self.on_step(self.chunks - 1, (slots, ranks, ntok), xs, ys)

    def _default_activations(self, T: int):
        import torch

        ex = self.executor
        pool = ex.pool
        if self._scratch is None:
            cap = ex.max_tokens
            self._scratch = (
                [[torch.zeros(cap, pool.h_in[g[0]], dtype=pool.dtype, device=pool.device) for g in ex.proj_groups]
                 for _ in range(pool.n_layers)],
                [[torch.zeros(cap, pool.h_out[p], dtype=pool.dtype, device=pool.device) for p in range(pool.n_proj)]
                 for _ in range(pool.n_layers)])
        xs, ys = self._scratch
        return [[x[:T] for x in row] for row in xs], [[y[:T] for y in row] for row in ys]


# --------------------------------------------------------------------------- decision replay
def replay_ops(cache, ops) -> list:
    """Drive `cache` (a fresh AdapterCache — ours or the reference's, duck-typed) through a
    recorded decision trace (`AdapterCache.op_log`) and return the ops whose outcome differs:
    return values (hit/miss + load bytes, eviction lists, prefetch candidates) and raised
    exceptions must be identical.  This is how a replica's hit/miss/evict decisions are
    checked against the reference AdapterCache fed that replica's sub-trace."""
    bad = []
    for i, rec in enumerate(ops):
        op, args = rec["op"], list(rec["args"])
        if op in ("evict_until", "set_capacity"):
            args[1] = set(args[1])
        fn = getattr(cache, op)
        try:
            ret = fn(*args)
        except Exception as ex:  # the reference's exception classes are its own
            if rec.get("raises") != type(ex).__name__:
                bad.append((i, op, rec.get("ret", rec.get("raises")), type(ex).__name__))
            continue
        if "raises" in rec:
            bad.append((i, op, rec["raises"], ret))
            continue
        if op == "acquire":
            ret = [ret.hit, ret.load_bytes]
        elif isinstance(ret, (list, tuple)):
            ret = list(ret)
        if ret != rec.get("ret"):
            bad.append((i, op, rec.get("ret"), ret))
    return bad


# --------------------------------------------------------------------------- replica loop
class ReplicaLoop:
    """One replica's serving loop over the device path (C4): the reference engine's admission
    and transfer transactions driven by real fills instead of simulated link time.

    Per step (`step(arrivals)`):
      1. transfer completions: every adapter whose fill finished (`cache.poll_fills()`, an
         event query — the host never blocks) gets finish_load + take_ref for each waiting
         request, which becomes ready (engine.py:294-301);
      2. admission, queued requests first then the step's arrivals (note_arrival,
         engine.py:288-291), up to `max_admit` per step: the memory check of try_admit
         (engine.py:497-506, against the replica's fixed capacity), acquire, set_capacity
         (engine.py:510); on a miss join the in-flight fill or evict_until + begin_load, which
         issues the pinned copy on the fill stream (engine.py:522-531); blocked and
         over-budget requests stay queued in arrival order;
      3. prefetch of the queued requests' adapters into free space (engine.py:457-470);
      4. the step: every ready request (hits and completed loads) runs one decode token
         through the executor (`run_batch(slots, ranks, ntok)`), after its fills on the device;
      5. every executed request releases its reference (engine.py:351-355).
    The cache's `op_log` is the replica's decision trace (replay_ops).
    """

    def __init__(self, cache, catalog, run_batch: Callable, capacity_tokens: int, step_us: int = 20_000,
                 prefetch: bool = True, record: bool = True, max_admit: Optional[int] = None):
        """max_admit: admissions per step (the scheduler's batch budget); requests beyond it
        stay queued in arrival order, and their adapters are the prefetch candidates."""
        self.cache = cache
        self.catalog = catalog
        self.run_batch = run_batch
        self.capacity = int(capacity_tokens)
        self.max_admit = max_admit
        self.step_us = int(step_us)
        self.prefetch = prefetch
        self.now = 0
        self.deferred: list[str] = []
        self.waiters: dict[str, int] = {}
        self.in_flight: set[str] = set()
        self.prefetched: set[str] = set()
        self._ordered: dict = {}
        if record:
            cache.op_log = []
        cache.set_capacity(self.capacity, set(), 0)
        self.stats = dict(steps=0, executed=0, hits=0, misses=0, joined=0, deferred=0, loads=0, prefetches=0,
                          prefetch_hits=0, completed=0)

    def _admit(self, aid: str, hints: set) -> Optional[bool]:
        """try_admit for one request: True ready now, False waiting on a fill, None blocked."""
        c = self.cache
        e = c.lookup(aid)
        ne_extra = 0 if ((e.resident and e.rc > 0) or e.loading) else e.size_tokens
        if c.non_evictable_tokens + ne_extra > self.capacity:
            return None
        res = c.acquire(aid, self.now)
        c.set_capacity(self.capacity, hints, self.now)
        if res.hit:
            self.stats["hits"] += 1
            if aid in self.prefetched:
                self.stats["prefetch_hits"] += 1
                self.prefetched.discard(aid)
            return True
        self.stats["misses"] += 1
        if aid in self.in_flight:
            self.stats["joined"] += 1
        else:
            c.evict_until(e.size_tokens, hints, self.now)
            c.begin_load(aid, self.now)
            self.in_flight.add(aid)
            self.stats["loads"] += 1
        self.waiters[aid] = self.waiters.get(aid, 0) + 1
        return False

    def step(self, arrivals) -> int:
        c = self.cache
        self.now += self.step_us
        now = self.now
        ready: list[str] = []
        # 1. completions
        for aid in c.poll_fills():
            if aid not in self.in_flight:
                continue
            self.in_flight.discard(aid)
            c.finish_load(aid, now)
            n = self.waiters.pop(aid, 0)
            for _ in range(n):
                c.take_ref(aid, now)
                ready.append(aid)
            if n == 0:
                self.prefetched.add(aid)
            self.stats["completed"] += 1
        # 2. admission (deferred first, in order)
        for aid in arrivals:
            c.note_arrival(aid, now)
        queue = self.deferred + list(arrivals)
        hints = set(queue)
        self.deferred = []
        admitted = 0
        for i, aid in enumerate(queue):
            if self.max_admit is not None and admitted >= self.max_admit:
                self.deferred.extend(queue[i:])
                break
            r = self._admit(aid, hints)
            if r is None:
                self.deferred.append(aid)
                continue
            admitted += 1
            if r:
                ready.append(aid)
        self.stats["deferred"] += len(self.deferred)
        # 3. prefetch for the still-queued adapters
        if self.prefetch and self.deferred:
            for aid in c.prefetch_candidates(list(dict.fromkeys(self.deferred)), c.free_tokens, now):
                if aid in self.in_flight:
                    continue
                c.begin_load(aid, now)
                self.in_flight.add(aid)
                self.stats["prefetches"] += 1
        # 4. the step's LoRA work, 5. release
        if ready:
            slots = np.array([c.slot_of(a) for a in ready], dtype=np.int32)
            ranks = np.array([self.catalog[a].rank for a in ready], dtype=np.int32)
            order_after_fills(c, ready, self._ordered)
            self.run_batch(slots, ranks, np.ones(len(ready), dtype=np.int32))
            for aid in ready:
                c.release(aid, now)
        self.stats["steps"] += 1
        self.stats["executed"] += len(ready)
        return len(ready)
