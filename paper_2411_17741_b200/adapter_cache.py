"""Adapter cache: the reference's insert / evict / lookup API, bit-exact, over a paged HBM pool.

`AdapterCache` restates the decision logic of the reference `adaptersim.adapter_cache`
(adapter_cache.py:65-328) with identical method names, arguments, return values, counters
and exceptions:

  lookup (90), free_tokens (93-95), non_evictable_tokens (97-103),
  resident_tokens_recount (105-109), acquire (111-121), take_ref (123-130),
  release (132-142), begin_load (144-151), finish_load (153-159), score (163-196),
  _eligible (198-202), _pick_victim (204-218), _evict (220-226), evict_until (228-248),
  set_capacity (250-263), note_arrival (267-271), prefetch_candidates (282-328).

Two host-side costs of the reference are removed without changing any decision
(SURVEY §8f row 4):
  * `non_evictable_tokens` is a running counter maintained at every state transition
    instead of an O(catalog) scan per admission attempt;
  * `_pick_victim` normalises the three features once per call (O(E)) instead of once per
    candidate (O(E^2)).  The float64 expressions are evaluated in the same order as the
    reference, so scores — and therefore victims — are bit-identical (tests/test_cache.py
    replays reference traces and compares every decision).

`PagedAdapterCache` adds the device side: each catalog adapter owns a fixed slot id, a
resident adapter owns ceil(rank/8) pages of an `AdapterPool`, `begin_load` issues the
pinned host->HBM fill on a side stream and `finish_load` is driven by its completion
event.  Page reuse after eviction waits on the compute stream's last-read event.
"""
from __future__ import annotations

import heapq
import math
from collections import deque
from dataclasses import dataclass, field
from typing import Iterable, Optional

from .model import AdapterSpec, CacheConfig, CachePolicy, PrefetchMode, TimePoint, enum_value


class InsufficientEvictableMemory(RuntimeError):
    """Even evicting every RC=0 entry cannot free the requested space."""


class CacheFault(AssertionError):
    """A cache operation violated a precondition (logic fault)."""


@dataclass
class AdapterEntry:
    """Residency + eviction metadata of one adapter (usage history survives eviction)."""

    spec: AdapterSpec
    last_used: TimePoint = 0
    rc: int = 0
    resident: bool = False
    loading: bool = False
    use_events: deque = field(default_factory=deque)

    @property
    def size_tokens(self) -> int:
        return self.spec.size_tokens

    def frequency(self, now: TimePoint, window_us: int) -> int:
        """Uses inside (now - window, now]; prunes older events (idempotent for fixed now)."""
        cutoff = now - window_us
        ev = self.use_events
        while ev and ev[0] <= cutoff:
            ev.popleft()
        return len(ev)


@dataclass(frozen=True)
class AcquireResult:
    hit: bool
    load_bytes: int = 0


_FIXED_WEIGHTS = {
    "lru": (0.0, 1.0, 0.0),
    "fairshare": (1 / 3, 1 / 3, 1 / 3),
}


def _jsonable(v):
    if isinstance(v, (set, frozenset)):
        return sorted(v)
    if isinstance(v, (list, tuple)):
        return list(v)
    return v


def _logged(name: str):
    """Record the call in `self.op_log` (when not None) as {"op", "args", "ret"} or
    {"op", "args", "raises"}: the replayable decision trace (serving.replay_ops, the format of
    tests/golden/cache_traces.json).  Iterable arguments are materialised first."""
    def deco(fn):
        def wrapped(self, *args):
            log = self.op_log
            if log is None:
                return fn(self, *args)
            if name == "prefetch_candidates":
                args = (list(args[0]),) + tuple(args[1:])
            rec = {"op": name, "args": [_jsonable(a) for a in args]}
            try:
                ret = fn(self, *args)
            except (InsufficientEvictableMemory, CacheFault) as ex:
                rec["raises"] = type(ex).__name__
                log.append(rec)
                raise
            rec["ret"] = [ret.hit, ret.load_bytes] if isinstance(ret, AcquireResult) else _jsonable(ret)
            log.append(rec)
            return ret
        wrapped.__name__, wrapped.__doc__, wrapped.__wrapped__ = fn.__name__, fn.__doc__, fn
        return wrapped
    return deco


def _pins(e: AdapterEntry) -> bool:
    """Counts toward non_evictable_tokens: in use by a running request, or in flight."""
    return (e.resident and e.rc > 0) or e.loading


class AdapterCache:
    """Adapter cache of one serving replica (single-threaded, synchronous transitions)."""

    def __init__(self, cfg: CacheConfig, catalog: dict[str, AdapterSpec]):
        self.cfg = cfg
        pol = enum_value(cfg.policy)
        self._policy = pol
        self.weights = _FIXED_WEIGHTS.get(pol, (cfg.weight_frequency, cfg.weight_recency, cfg.weight_size))
        self.entries = {aid: AdapterEntry(spec) for aid, spec in catalog.items()}
        self.capacity_tokens = 0
        self.used_tokens = 0
        self.hits = 0
        self.misses = 0
        self.evictions = 0
        self.loads = 0
        self._arrivals: dict[str, deque] = {}
        self._pinned_tokens = 0
        self.op_log: Optional[list] = None  # set to [] to record the decision trace
        self._log2 = {aid: math.log2(spec.size_tokens) for aid, spec in catalog.items()}

    # -- residency and reference counting ------------------------------------------------
    def lookup(self, adapter_id: str) -> AdapterEntry:
        return self.entries[adapter_id]

    @property
    def free_tokens(self) -> int:
        return self.capacity_tokens - self.used_tokens

    @property
    def non_evictable_tokens(self) -> int:
        return self._pinned_tokens

    def non_evictable_tokens_recount(self) -> int:
        return sum(e.size_tokens for e in self.entries.values() if _pins(e))

    def resident_tokens_recount(self) -> int:
        return sum(e.size_tokens for e in self.entries.values() if e.resident or e.loading)

    def _transition(self, e: AdapterEntry, before: bool) -> None:
        after = _pins(e)
        if after != before:
            self._pinned_tokens += e.size_tokens if after else -e.size_tokens

    @_logged("acquire")
    def acquire(self, adapter_id: str, now: TimePoint) -> AcquireResult:
        e = self.entries[adapter_id]
        if not e.resident:
            self.misses += 1
            return AcquireResult(hit=False, load_bytes=e.spec.size_bytes)
        before = _pins(e)
        e.rc += 1
        e.last_used = now
        e.use_events.append(now)
        self.hits += 1
        self._transition(e, before)
        return AcquireResult(hit=True)

    @_logged("take_ref")
    def take_ref(self, adapter_id: str, now: TimePoint) -> None:
        e = self.entries[adapter_id]
        if not e.resident:
            raise CacheFault(f"take_ref on non-resident adapter {adapter_id}")
        before = _pins(e)
        e.rc += 1
        e.last_used = now
        e.use_events.append(now)
        self._transition(e, before)

    @_logged("release")
    def release(self, adapter_id: str, now: TimePoint) -> None:
        e = self.entries[adapter_id]
        if e.rc < 1:
            raise CacheFault(f"release on adapter {adapter_id} with RC=0")
        before = _pins(e)
        e.rc -= 1
        if e.rc == 0 and self._policy == "none":
            e.resident = False
            self.used_tokens -= e.size_tokens
            self._on_drop(e)
        self._transition(e, before)

    @_logged("begin_load")
    def begin_load(self, adapter_id: str, now: TimePoint) -> None:
        e = self.entries[adapter_id]
        if e.resident or e.loading:
            raise CacheFault(f"begin_load on already-present adapter {adapter_id}")
        before = _pins(e)
        e.loading = True
        self.used_tokens += e.size_tokens
        self.loads += 1
        self._transition(e, before)
        self._on_begin_load(e)

    @_logged("finish_load")
    def finish_load(self, adapter_id: str, now: TimePoint) -> None:
        e = self.entries[adapter_id]
        if not e.loading:
            raise CacheFault(f"finish_load without begin_load for {adapter_id}")
        before = _pins(e)
        e.loading = False
        e.resident = True
        e.last_used = now
        self._transition(e, before)

    # -- scoring and eviction --------------------------------------------------------------
    def score(self, entry: AdapterEntry, candidates: list[AdapterEntry], now: TimePoint,
              weights: Optional[tuple[float, float, float]] = None) -> float:
        """wf*norm(freq) + wr*norm(last_used) + ws*norm(log2 size), min-max over candidates,
        an all-equal feature normalising to 1 (adapter_cache.py:163-196)."""
        window = self.cfg.frequency_window_us
        freqs = [c.frequency(now, window) for c in candidates]
        recs = [c.last_used for c in candidates]
        sizes = [math.log2(c.size_tokens) for c in candidates]
        bounds = ((min(freqs), max(freqs)), (min(recs), max(recs)), (min(sizes), max(sizes)))
        return self._score_with(entry.frequency(now, window), entry.last_used,
                                math.log2(entry.size_tokens), bounds, weights or self.weights)

    @staticmethod
    def _score_with(freq, rec, size, bounds, weights) -> float:
        (flo, fhi), (rlo, rhi), (slo, shi) = bounds
        wf, wr, ws = weights
        nf = 1.0 if fhi == flo else (freq - flo) / (fhi - flo)
        nr = 1.0 if rhi == rlo else (rec - rlo) / (rhi - rlo)
        ns = 1.0 if shi == slo else (size - slo) / (shi - slo)
        return wf * nf + wr * nr + ws * ns

    def _eligible(self) -> list[AdapterEntry]:
        return [e for e in self.entries.values() if e.resident and e.rc == 0 and not e.loading]

    def _pick_victim(self, hints: set[str], now: TimePoint) -> Optional[AdapterEntry]:
        """Lowest (score, size_tokens, adapter_id) in the unhinted tier, else among all
        eligible entries; features normalised once over the eligible set."""
        eligible = self._eligible()
        if not eligible:
            return None
        window = self.cfg.frequency_window_us
        freqs = [e.frequency(now, window) for e in eligible]
        recs = [e.last_used for e in eligible]
        sizes = [self._log2.get(e.spec.adapter_id) or math.log2(e.size_tokens) for e in eligible]
        bounds = ((min(freqs), max(freqs)), (min(recs), max(recs)), (min(sizes), max(sizes)))
        tier = [i for i, e in enumerate(eligible) if e.spec.adapter_id not in hints]
        if not tier:
            tier = range(len(eligible))
        best, best_key = None, None
        w = self.weights
        for i in tier:
            e = eligible[i]
            key = (self._score_with(freqs[i], recs[i], sizes[i], bounds, w), e.size_tokens, e.spec.adapter_id)
            if best_key is None or key < best_key:
                best, best_key = e, key
        return best

    def _evict(self, entry: AdapterEntry) -> str:
        if entry.rc != 0 or entry.loading:
            raise CacheFault(f"attempted to evict in-use adapter {entry.spec.adapter_id}")
        before = _pins(entry)
        entry.resident = False
        self.used_tokens -= entry.size_tokens
        self.evictions += 1
        self._transition(entry, before)
        self._on_drop(entry)
        return entry.spec.adapter_id

    @_logged("evict_until")
    def evict_until(self, needed_tokens: int, hints: set[str], now: TimePoint) -> list[str]:
        """Evict victims until free >= needed; atomic InsufficientEvictableMemory otherwise."""
        if self.free_tokens >= needed_tokens:
            return []
        evictable = sum(e.size_tokens for e in self._eligible())
        if self.free_tokens + evictable < needed_tokens:
            raise InsufficientEvictableMemory(
                f"need {needed_tokens} tokens, only {self.free_tokens + evictable} freeable")
        out = []
        while self.free_tokens < needed_tokens:
            out.append(self._evict(self._pick_victim(hints, now)))
        return out

    @_logged("set_capacity")
    def set_capacity(self, tokens: int, hints: set[str], now: TimePoint) -> list[str]:
        """Shrink to `tokens` by eviction; capacity never drops below in-use occupancy."""
        out = []
        while self.used_tokens > tokens:
            victim = self._pick_victim(hints, now)
            if victim is None:
                break
            out.append(self._evict(victim))
        self.capacity_tokens = max(tokens, self.used_tokens)
        return out

    # -- prefetch ---------------------------------------------------------------------------
    @_logged("note_arrival")
    def note_arrival(self, adapter_id: str, now: TimePoint) -> None:
        if enum_value(self.cfg.prefetch) != PrefetchMode.HISTOGRAM.value:
            return
        self._arrivals.setdefault(adapter_id, deque()).append(now)

    def _arrival_count(self, adapter_id: str, now: TimePoint) -> int:
        ev = self._arrivals.get(adapter_id)
        if not ev:
            return 0
        cutoff = now - self.cfg.frequency_window_us
        while ev and ev[0] <= cutoff:
            ev.popleft()
        return len(ev)

    @_logged("prefetch_candidates")
    def prefetch_candidates(self, queued_adapter_ids: Iterable[str], free_tokens: int,
                            now: TimePoint) -> list[str]:
        """Queue-driven greedy fit; histogram mode adds top window-arrival adapters."""
        mode = enum_value(self.cfg.prefetch)
        if mode == PrefetchMode.OFF.value:
            return []
        chosen: list[str] = []
        taken: set[str] = set()
        budget = free_tokens
        queued = list(queued_adapter_ids)
        for aid in queued:
            e = self.entries[aid]
            if e.resident or e.loading or aid in taken:
                continue
            if e.size_tokens <= budget:
                chosen.append(aid)
                taken.add(aid)
                budget -= e.size_tokens
        if mode == PrefetchMode.HISTOGRAM.value:
            qset = set(queued)
            ranked = sorted(
                ((self._arrival_count(aid, now), aid) for aid, e in self.entries.items()
                 if not e.resident and not e.loading and aid not in taken and aid not in qset),
                key=lambda pr: (-pr[0], pr[1]))
            for count, aid in ranked:
                if count == 0:
                    break
                size = self.entries[aid].size_tokens
                if size <= budget:
                    chosen.append(aid)
                    taken.add(aid)
                    budget -= size
        return chosen

    # -- hooks for the paged subclass --------------------------------------------------------
    def _on_begin_load(self, entry: AdapterEntry) -> None:
        pass

    def _on_drop(self, entry: AdapterEntry) -> None:
        pass


class PagedAdapterCache(AdapterCache):
    """AdapterCache whose resident set lives in an AdapterPool (pages of 8 rank rows).

    Token accounting is the reference's (size_tokens = 4 * rank); a page holds 8 rank rows
    = 32 tokens.  The constructor requires every catalog adapter's size_tokens to equal its
    page count x 32 (ranks that are multiples of 8 under the default byte model), and
    set_capacity caps the capacity at pool.n_pages x 32, so the page allocator can never
    contradict a token-level decision.

    host_store: adapter_id -> packed pinned host tensor (AdapterPool.pack_host); the
    reference's host-memory adapter repository.  fill_stream: side stream for miss fills.
    compute_stream: stream lora_apply runs on (page reuse waits on its events).
    """

    TOKENS_PER_PAGE = 32

    def __init__(self, cfg: CacheConfig, catalog: dict[str, AdapterSpec], pool, host_store=None,
                 fill_stream=None, compute_stream=None, event_factory=None):
        """event_factory(stream) -> an event recorded on `stream` (default torch.cuda.Event)."""
        super().__init__(cfg, catalog)
        import torch

        self._torch = torch
        self._record = event_factory or self._record_cuda
        self.pool = pool
        if len(catalog) > pool.n_slots:
            raise ValueError(f"pool has {pool.n_slots} slots for a catalog of {len(catalog)} adapters")
        bad = [aid for aid, spec in catalog.items()
               if spec.size_tokens != -(-spec.rank // 8) * self.TOKENS_PER_PAGE]
        if bad:
            raise ValueError(f"page and token accounting disagree for {len(bad)} adapters (e.g. {bad[0]}): "
                             "size_tokens must equal ceil(rank/8) * 32 (ranks multiples of 8)")
        self.slot_ids = {aid: i for i, aid in enumerate(catalog)}
        self.host_store = host_store if host_store is not None else {}
        self.fill_stream = fill_stream or torch.cuda.Stream(device=pool.device)
        self.compute_stream = compute_stream or torch.cuda.current_stream(pool.device)
        self._free_pages = list(range(pool.n_pages))
        heapq.heapify(self._free_pages)
        self._page_release: dict[int, object] = {}
        self._slot_release: dict[int, object] = {}
        self._fill_events: dict[str, object] = {}
        self.fill_bytes = 0
        self.fill_count = 0

    def _record_cuda(self, stream):
        ev = self._torch.cuda.Event()
        ev.record(stream)
        return ev

    # -- slots / pages -----------------------------------------------------------------------
    def slot_of(self, adapter_id: str) -> int:
        return self.slot_ids[adapter_id]

    def pages_of(self, adapter_id: str) -> list[int]:
        return list(self.pool.slot_pages[self.slot_ids[adapter_id]])

    @property
    def max_capacity_tokens(self) -> int:
        return self.pool.n_pages * self.TOKENS_PER_PAGE

    def set_capacity(self, tokens: int, hints: set[str], now: TimePoint) -> list[str]:
        """The reference's set_capacity (adapter_cache.py:250-263) with the target capped at
        the pool's physical size (n_pages x 32 tokens)."""
        return super().set_capacity(min(int(tokens), self.max_capacity_tokens), hints, now)

    def begin_load(self, adapter_id: str, now: TimePoint) -> None:
        """The reference's begin_load (adapter_cache.py:144-151); the page check runs before any
        state changes, so a CacheFault for lack of pages leaves the cache untouched."""
        e = self.entries[adapter_id]
        if not (e.resident or e.loading):
            n = -(-e.spec.rank // 8)
            if len(self._free_pages) < n:
                raise CacheFault(f"no free pool pages for {adapter_id} (need {n}, {len(self._free_pages)} free)")
        super().begin_load(adapter_id, now)

    def _on_begin_load(self, entry: AdapterEntry) -> None:
        aid = entry.spec.adapter_id
        rank = entry.spec.rank
        n = -(-rank // 8)
        pages = sorted(heapq.heappop(self._free_pages) for _ in range(n))
        fs = self.fill_stream
        slot = self.slot_ids[aid]
        ev = self._slot_release.pop(slot, None)
        if ev is not None:
            fs.wait_event(ev)  # the slot's unbind (compute stream) lands before this rebind
        for p in pages:
            ev = self._page_release.pop(p, None)
            if ev is not None:
                fs.wait_event(ev)  # a kernel launched before the eviction may still read p
        self.pool.set_slot(slot, rank, pages, stream=fs)
        src = self.host_store.get(aid)
        if src is not None:
            self.pool.fill_async(slot, src, stream=fs)
            self.fill_bytes += src.numel()
            self.fill_count += 1
        self._fill_events[aid] = self._record(fs)

    def _on_drop(self, entry: AdapterEntry) -> None:
        aid = entry.spec.adapter_id
        slot = self.slot_ids[aid]
        pages = self.pool.slot_pages[slot]
        # unbind first, then record: the event covers every kernel that read the pages AND the
        # unbind itself, so a later rebind of this slot or reuse of these pages (fill stream,
        # which waits on it) is ordered after both
        self.pool.set_slot(slot, 0, [], stream=self.compute_stream)
        ev = self._record(self.compute_stream)
        self._slot_release[slot] = ev
        for p in pages:
            self._page_release[p] = ev
            heapq.heappush(self._free_pages, p)
        self._fill_events.pop(aid, None)

    def fill_event(self, adapter_id: str):
        """Completion event of the adapter's last fill (None if never filled)."""
        return self._fill_events.get(adapter_id)

    def poll_fills(self) -> list[str]:
        """Adapters whose fill completed (event query), in ascending id order; the engine
        calls finish_load for these (engine.py:294-301 `_on_transfer_complete`)."""
        done = [aid for aid, ev in self._fill_events.items()
                if self.entries[aid].loading and ev.query()]
        return sorted(done)

    def wait_ready(self, adapter_ids: Iterable[str], stream=None) -> None:
        """Make `stream` (default compute) wait for the fills of these adapters."""
        s = stream or self.compute_stream
        for aid in adapter_ids:
            ev = self._fill_events.get(aid)
            if ev is not None:
                s.wait_event(ev)
