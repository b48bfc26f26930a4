"""PagedAdapterCache host logic on CPU (fake pool and streams; no GPU): the page/token
accounting guard, the set_capacity cap, atomic begin_load, and the stream ordering of an
eviction followed by a reload of the same adapter (the unbind must precede the rebind).

Reference: AdapterCache.begin_load / set_capacity / _evict (adapter_cache.py:144-151,
220-226, 250-263); the paged subclass adds the device side."""
import pytest

from paper_2411_17741_b200.adapter_cache import CacheFault, PagedAdapterCache
from paper_2411_17741_b200.model import CacheConfig, make_adapter_spec


class _Log(list):
    pass


class _Event:
    def __init__(self, log, stream):
        self.stream = stream
        self.id = len([x for x in log if x[0] == "record"])
        log.append(("record", stream.name, self.id))

    def query(self):
        return True


class _Stream:
    def __init__(self, name, log):
        self.name, self.log = name, log

    def wait_event(self, ev):
        self.log.append(("wait", self.name, ev.id))


class _Pool:
    def __init__(self, n_pages, n_slots, log):
        self.n_pages, self.n_slots, self.log = n_pages, n_slots, log
        self.slot_pages = [[] for _ in range(n_slots)]
        self.device = "cpu"

    def set_slot(self, slot, rank, pages, stream=None):
        self.log.append(("set_slot", stream.name, slot, rank, tuple(pages)))
        self.slot_pages[slot] = list(pages)

    def fill_async(self, slot, src, stream=None):
        self.log.append(("fill", stream.name, slot))


def _cache(ranks, n_pages, log=None):
    log = log if log is not None else _Log()
    catalog = {f"a{i}": make_adapter_spec(f"a{i}", r) for i, r in enumerate(ranks)}
    pool = _Pool(n_pages, len(catalog), log)
    c = PagedAdapterCache(CacheConfig(), catalog, pool, host_store={},
                          fill_stream=_Stream("fill", log), compute_stream=_Stream("compute", log),
                          event_factory=lambda s: _Event(log, s))
    return c, log


def test_rejects_ranks_whose_pages_and_tokens_disagree():
    with pytest.raises(ValueError, match="page and token accounting"):
        _cache([8, 12], 8)  # rank 12: 48 tokens but 2 pages = 64 tokens


def test_set_capacity_is_capped_at_the_pool():
    c, _ = _cache([8, 16], 3)
    c.set_capacity(10_000, set(), 0)
    assert c.capacity_tokens == 3 * 32


def test_begin_load_without_pages_is_atomic():
    c, _ = _cache([64, 16], 9)  # 8 + 2 pages > 9
    c.set_capacity(10_000, set(), 0)  # capped: 288 tokens
    c.begin_load("a0", 1)
    before = (c.used_tokens, c.loads, c.non_evictable_tokens, c.lookup("a1").loading)
    with pytest.raises(CacheFault, match="no free pool pages"):
        c.begin_load("a1", 2)
    assert (c.used_tokens, c.loads, c.non_evictable_tokens, c.lookup("a1").loading) == before


def test_evict_then_reload_orders_unbind_before_rebind():
    c, log = _cache([16, 16], 2)
    c.set_capacity(64, set(), 0)
    c.begin_load("a0", 1)
    c.finish_load("a0", 2)
    assert c.evict_until(32, set(), 3) == ["a0"]  # capacity 64, a0 holds 32: a1 needs its room
    c.begin_load("a1", 4)  # reuses a0's pages
    c.finish_load("a1", 5)
    assert c.evict_until(64, set(), 6) == ["a1"]
    c.begin_load("a0", 7)  # a0 again: same slot, pages released by a1's eviction
    i_unbind = log.index(("set_slot", "compute", 0, 0, ()))
    ev_after_unbind = next(x for x in log[i_unbind:] if x[0] == "record" and x[1] == "compute")
    # the release event of a0's eviction is recorded after its unbind ...
    assert log.index(ev_after_unbind) > i_unbind
    # ... and the fill stream waits on it before rebinding slot 0
    rebinds = [i for i, x in enumerate(log) if x[0] == "set_slot" and x[2] == 0 and x[3] > 0]
    i_rebind = rebinds[-1]
    waits = [i for i, x in enumerate(log[:i_rebind]) if x == ("wait", "fill", ev_after_unbind[2])]
    assert waits, log
    # a1's pages (released by its own eviction) are also waited on before the rebind
    i_unbind1 = log.index(("set_slot", "compute", 1, 0, ()))
    ev1 = next(x for x in log[i_unbind1:] if x[0] == "record")
    assert ("wait", "fill", ev1[2]) in log[:i_rebind]
