"""Engine seams on the CPU: the device path (PagedAdapterCache + step executor, with fake
pool/streams) installed into the UNMODIFIED reference engine must leave every engine
decision unchanged — `simulate()` returns a byte-identical RunResult / records CSV
(reference determinism test: test_engine.py:195-202) — while every miss and prefetch
issues exactly one fill, every transfer-complete event is gated on its fill, and every
step's batch is executed with all of its adapters bound to pages.

Seams: engine.py:160 (cache), 294-301 (_on_transfer_complete), 443-455 (_try_schedule ->
step_duration), 457-470 (_issue_prefetches), 491-532 (_Oracle.try_admit)."""
import pytest

from _fakes import Executor, paged_cache
from paper_2411_17741_b200.serving import EngineSeams, SeamError

pytestmark = pytest.mark.reference


def _cfg(ref, policy="mlq", cache="cost-aware", prefetch="off", seed=3, slots=9000, rate=1.0, dur=120.0):
    from adaptersim.model import config_from_dict

    return config_from_dict({
        "workload": {"arrival_rate": rate, "duration_s": dur, "seed": seed},
        "scheduler": {"policy": policy, "refresh_us": 20_000_000},
        "cache": {"policy": cache, "prefetch": prefetch},
        "hardware": {"total_token_slots": slots, "link_bandwidth_bytes_per_sec": 100_000_000},
    })


def _csv(records, path):
    from adaptersim.metrics import write_records_csv

    write_records_csv(records, str(path))
    return path.read_bytes()


CASES = [
    dict(policy="mlq", cache="cost-aware", prefetch="off"),
    dict(policy="mlq", cache="cost-aware", prefetch="queue-driven"),
    dict(policy="fifo", cache="lru", prefetch="histogram"),
    dict(policy="sjf", cache="fairshare", prefetch="off", seed=5),
    dict(policy="mlq", cache="none", prefetch="off", seed=7),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(str(v) for v in c.values()))
@pytest.mark.parametrize("fill_wait", ["stream", "poll"])
def test_installed_seams_leave_run_result_byte_identical(reference_pkg, tmp_path, case, fill_wait):
    from adaptersim.engine import Simulation, simulate

    cfg = _cfg(reference_pkg, **case)
    want = simulate(cfg)

    sim = Simulation(_cfg(reference_pkg, **case))
    n_pages = cfg.hardware.total_token_slots // 32 + 1
    cache, log = paged_cache(sim.cfg.cache, sim.catalog, n_pages)
    ex = Executor(cache.pool)
    seams = EngineSeams(cache, ex, activations=lambda T: (None, None), fill_wait=fill_wait).install(sim)
    got = sim.run()

    assert got == want  # every record, counter, snapshot and occupancy figure
    assert _csv(got.records, tmp_path / "a.csv") == _csv(want.records, tmp_path / "b.csv")
    # every transfer the engine modelled was a real fill, and each completed through the seam
    fills = [x for x in log if x[0] == "fill"]
    assert len(fills) == want.transfer_count == cache.loads
    assert seams.transfers_completed == want.transfer_count
    assert seams.steps == want.steps
    # every step's requests were executed (decoders 1 token, prefills input_tokens)
    assert sum(sum(c[2]) for c in ex.chunks) == seams.tokens > 0
    assert all(sum(c[2]) <= ex.max_tokens for c in ex.chunks)


def test_fill_precedes_rebind_and_step_orders_after_fill(reference_pkg):
    """Device stream order of the miss transaction: set_slot + fill on the fill stream, the
    fill's event recorded after the copy, and the compute stream waits on it before the
    first step that reads the adapter."""
    from adaptersim.engine import Simulation

    sim = Simulation(_cfg(reference_pkg, slots=9000, dur=40.0))
    cache, log = paged_cache(sim.cfg.cache, sim.catalog, 9000 // 32 + 1)
    ex = Executor(cache.pool)
    uploads = []
    orig = ex.upload

    def upload(slots, ranks, ntok, stream=None):
        uploads.append(len(log))
        log.append(("upload",))
        return orig(slots, ranks, ntok, stream)

    ex.upload = upload
    EngineSeams(cache, ex, activations=lambda T: (None, None)).install(sim)
    sim.run()
    # for every fill: its record follows it on the fill stream, and a compute-stream wait on
    # that record precedes the first upload after it
    for i, x in enumerate(log):
        if x[0] != "fill":
            continue
        rec = next(y for y in log[i + 1:] if y[0] == "record" and y[1] == "fill")
        j = log.index(rec)
        nxt_upload = next((k for k in uploads if k > j), None)
        if nxt_upload is None:
            continue
        waits = [y for y in log[j:nxt_upload] if y[0] == "wait" and y[1] == "compute" and y[2] == rec[2]]
        slot = x[2]
        # the step right after this fill reads the slot only if the engine scheduled it; then the wait exists
        reads = any(slot in c[0] for c in ex.chunks[uploads.index(nxt_upload):uploads.index(nxt_upload) + 1])
        assert waits or not reads


def test_install_rejects_foreign_catalog_and_running_sim(reference_pkg):
    from adaptersim.engine import Simulation

    from paper_2411_17741_b200.model import CacheConfig, make_adapter_spec

    sim = Simulation(_cfg(reference_pkg, dur=10.0))
    cache, _ = paged_cache(CacheConfig(), {"r8-0": make_adapter_spec("r8-0", 8)}, 4)
    with pytest.raises(SeamError, match="catalog"):
        EngineSeams(cache).install(sim)


def test_step_with_unloaded_adapter_is_a_seam_error():
    from paper_2411_17741_b200.model import CacheConfig, make_adapter_spec

    cat = {"r8-0": make_adapter_spec("r8-0", 8)}
    cache, _ = paged_cache(CacheConfig(), cat, 4)
    seams = EngineSeams(cache, Executor(cache.pool), activations=lambda T: (None, None))

    class R:
        class spec:
            adapter_id = "r8-0"
            input_tokens = 5

    with pytest.raises(SeamError, match="not resident"):
        seams.run_step([R()], [], {"r8-0": 8})
