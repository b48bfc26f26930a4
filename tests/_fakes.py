"""CPU stand-ins for the device objects PagedAdapterCache and the engine seams touch (pool,
streams, events, step executor), so the host logic runs in the CPU suite.  Every call is
logged in order, which lets tests check the stream ordering the device would see."""
from __future__ import annotations


class Log(list):
    pass


class Event:
    delay = 0  # queries before a fill-stream event reports completion (simulated copy time)

    def __init__(self, log, stream):
        self.stream = stream
        self.id = len([x for x in log if x[0] == "record"])
        self.left = Event.delay if stream.name == "fill" else 0
        self.done = self.left == 0
        log.append(("record", stream.name, self.id))

    def query(self):
        if not self.done:
            self.left -= 1
            self.done = self.left <= 0
        return self.done

    def synchronize(self):
        self.done = True


class Stream:
    def __init__(self, name, log):
        self.name, self.log = name, log

    def wait_event(self, ev):
        self.log.append(("wait", self.name, ev.id))


class Pool:
    def __init__(self, n_pages, n_slots, log, n_layers=1, h=64):
        self.n_pages, self.n_slots, self.log = n_pages, n_slots, log
        self.slot_pages = [[] for _ in range(n_slots)]
        self.device = "cpu"
        self.n_layers, self.h_in, self.h_out, self.n_proj = n_layers, [h], [h], 1

    def set_slot(self, slot, rank, pages, stream=None):
        self.log.append(("set_slot", stream.name, slot, rank, tuple(pages)))
        self.slot_pages[slot] = list(pages)

    def fill_async(self, slot, src, stream=None):
        self.log.append(("fill", stream.name, slot))


class Executor:
    """Records every uploaded chunk; run() is a no-op (the pool's pages are checked instead)."""

    def __init__(self, pool, max_tokens=4096):
        self.pool, self.max_tokens, self.proj_groups = pool, max_tokens, [[0]]
        self.chunks = []

    def upload(self, slots, ranks, ntok, stream=None):
        self.chunks.append((list(map(int, slots)), list(map(int, ranks)), list(map(int, ntok))))
        # every slot the step reads is bound to pages at this point in stream order
        for s in slots:
            assert self.pool.slot_pages[int(s)], f"slot {int(s)} unbound at upload"
        return int(sum(ntok))

    def run(self, xs, ys, stream=None):
        pass


def paged_cache(cfg, catalog, n_pages, log=None):
    from paper_2411_17741_b200.adapter_cache import PagedAdapterCache

    log = log if log is not None else Log()
    pool = Pool(n_pages, len(catalog), log)
    c = PagedAdapterCache(cfg, catalog, pool, host_store={a: _Src() for a in catalog},
                          fill_stream=Stream("fill", log), compute_stream=Stream("compute", log),
                          event_factory=lambda s: Event(log, s))
    return c, log


class _Src:
    def numel(self):
        return 1
