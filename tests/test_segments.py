"""Segment tables and the batch-descriptor seam (CPU).

* The numpy oracle's canonical table on every step captured from the reference simulate()
  (tests/golden/sim_batches.json): Σ rank x tokens over segments equals the reference's
  own adapter_units for that step (engine.py:64-76), tokens are a permutation, segments
  sorted by slot with batch order kept inside a slot.
* executor.batch_arrays on the (prefills, decoders) tuple and on BatchResult.admitted.
"""
import json
from types import SimpleNamespace

import numpy as np
import pytest

from oracle.segments_ref import adapter_units as units_ref
from oracle.segments_ref import build_segments_ref
from paper_2411_17741_b200.executor import adapter_units, batch_arrays
from paper_2411_17741_b200.workload import rank_of_id


def _req(aid, ntok=1):
    return SimpleNamespace(spec=SimpleNamespace(adapter_id=aid, input_tokens=ntok))


def _step_batch(step):
    return ([_req(a, n) for a, n in step["prefills"]], [_req(a) for a in step["decoders"]])


@pytest.fixture(scope="module")
def sim_steps(golden_dir):
    return json.loads((golden_dir / "sim_batches.json").read_text())["steps"]


def _slot_of_factory():
    table = {}

    def slot_of(aid):
        # distinct slots in a scrambled (not first-seen) order
        return table.setdefault(aid, (len(table) * 37) % 1009)

    return slot_of


def check_table(req_slot, req_rank, req_ntok, perm, seg_off, seg_slot, seg_rank):
    n = len(req_slot)
    tok_off = np.concatenate([[0], np.cumsum(req_ntok)])
    valid = [i for i in range(n) if req_slot[i] >= 0]
    assert seg_off[0] == 0 and seg_off[-1] == len(perm) == sum(req_ntok[i] for i in valid)
    assert np.all(np.diff(seg_slot) > 0)  # one segment per distinct slot, ascending
    assert len(set(perm.tolist())) == len(perm)
    for s in range(len(seg_slot)):
        rows = perm[seg_off[s]:seg_off[s + 1]]
        owners = [int(np.searchsorted(tok_off, t, side="right") - 1) for t in rows]
        assert all(req_slot[o] == seg_slot[s] and req_rank[o] == seg_rank[s] for o in owners)
        assert owners == sorted(owners)  # batch order inside a slot
        assert list(rows) == sorted(rows)


def test_sim_batches_units_match_reference(sim_steps):
    assert len(sim_steps) >= 200
    n_prefill_steps = 0
    for st in sim_steps:
        batch = _step_batch(st)
        slots, ranks, ntok = batch_arrays(batch, _slot_of_factory(), rank_of_id)
        assert adapter_units(batch, rank_of_id) == st["adapter_units"]
        perm, seg_off, seg_slot, seg_rank = build_segments_ref(slots, ranks, ntok)
        check_table(slots, ranks, ntok, perm, seg_off, seg_slot, seg_rank)
        seg_units = int(np.sum(np.diff(seg_off).astype(np.int64) * seg_rank))
        assert seg_units == st["adapter_units"] == units_ref(ranks, ntok)
        n_prefill_steps += bool(st["prefills"])
    assert n_prefill_steps > 0


def test_no_adapter_rows_and_empty_batch():
    perm, seg_off, seg_slot, seg_rank = build_segments_ref([3, -1, 3, 0], [8, 0, 8, 16], [2, 5, 1, 3])
    assert perm.tolist() == [8, 9, 10, 0, 1, 7]
    assert seg_off.tolist() == [0, 3, 6] and seg_slot.tolist() == [0, 3] and seg_rank.tolist() == [16, 8]
    perm, seg_off, seg_slot, seg_rank = build_segments_ref([], [], [])
    assert len(perm) == 0 and seg_off.tolist() == [0] and len(seg_slot) == 0


def test_zero_token_requests_are_empty():
    perm, seg_off, seg_slot, _ = build_segments_ref([1, 2, 1], [8, 8, 8], [0, 2, 1])
    assert perm.tolist() == [2, 0, 1] and seg_off.tolist() == [0, 1, 3] and seg_slot.tolist() == [1, 2]


def test_batch_arrays_on_admitted_lists(golden_dir):
    """BatchResult.admitted (scheduler.py:246-255; fixture from the reference
    generate_batch) enters as prefills with input_tokens each."""
    results = json.loads((golden_dir / "batch_results.json").read_text())
    seen = 0
    for res in results:
        assert sum(res["consumed"]) + res["leftover"] + sum(res["stranded"]) == sum(res["budgets"])
        admitted = [_req(aid, n) for _rid, aid, n in res["admitted"]]
        slots, ranks, ntok = batch_arrays(admitted, lambda a: int(a.split("-")[1]), rank_of_id)
        assert ntok.tolist() == [n for _, _, n in res["admitted"]]
        assert ranks.tolist() == [rank_of_id(a) for _, a, _ in res["admitted"]]
        seen += len(admitted)
    assert seen > 0


def test_batch_arrays_order_prefills_then_decoders():
    b = ([_req("r8-0", 5), _req("r16-1", 3)], [_req("r8-0"), _req("r128-2")])
    slots, ranks, ntok = batch_arrays(b, {"r8-0": 0, "r16-1": 1, "r128-2": 2}.__getitem__, rank_of_id)
    assert slots.tolist() == [0, 1, 0, 2] and ranks.tolist() == [8, 16, 8, 128] and ntok.tolist() == [5, 3, 1, 1]
    assert adapter_units(b, rank_of_id) == 8 * 5 + 16 * 3 + 8 + 128


@pytest.mark.reference
def test_live_step_duration_lora_term(reference_pkg, sim_steps):
    """The reference's LoRA seam (engine.py:67-77) is coef x adapter_units: the same batch
    with its ranks and with all ranks zero differs by that term (integer µs rounding)."""
    from adaptersim import engine, model

    params = model.CostModelParams()
    cm = engine.CostModel(params)
    coef = params.adapter_compute_per_rank_token_us
    for st in sim_steps[:100]:
        pre = [SimpleNamespace(spec=SimpleNamespace(adapter_id=a, input_tokens=n), tokens_generated=0)
               for a, n in st["prefills"]]
        dec = [SimpleNamespace(spec=SimpleNamespace(adapter_id=a, input_tokens=1), tokens_generated=0)
               for a in st["decoders"]]
        ranks = {a: rank_of_id(a) for a in [a for a, _ in st["prefills"]] + st["decoders"]}
        with_lora = cm.step_duration(pre, dec, ranks)
        without = cm.step_duration(pre, dec, {a: 0 for a in ranks})
        assert abs((with_lora - without) - coef * st["adapter_units"]) <= 1.0


def test_segment_token_bounds_route_hints():
    """Host routing hints (executor.segment_token_bounds): one segment per distinct slot,
    min/max of their token counts; a rank above the tcgen05 limit forces min = 0."""
    from paper_2411_17741_b200.executor import segment_token_bounds
    from oracle.segments_ref import build_segments_ref

    slots = [3, 1, 3, -1, 7, 1]
    ranks = [16, 8, 16, 0, 64, 8]
    ntok = [100, 1, 40, 9, 70, 2]
    perm, off, sl, rk = build_segments_ref(slots, ranks, ntok)
    lens = [int(off[i + 1] - off[i]) for i in range(len(sl)) if sl[i] >= 0]
    assert segment_token_bounds(slots, ranks, ntok) == (min(lens), max(lens)) == (3, 140)
    assert segment_token_bounds(slots, [16, 8, 16, 0, 256, 8], ntok) == (0, 140)
    assert segment_token_bounds([-1, -1], [0, 0], [5, 5]) == (0, 0)


def test_multiqueue_batch_descriptor_pinned(golden_dir):
    """MultiQueueScheduler.generate_batch (scheduler.py:528-550), from the reference: Algorithm
    1's admission order on the reference test's hand trace (test_scheduler.py:222-232: needs
    [30, 30, 30, 40, 50, 30], consumed [120, 40, 50], leftover 30; the implementation's
    stranded ledger is [10, 0, 50]) and the budget conservation on every MLQ case; the
    admitted list is the batch the segment builder consumes, in that order."""
    results = json.loads((golden_dir / "batch_results.json").read_text())
    mlq = [r for r in results if r["scheduler"] == "mlq"]
    assert len(mlq) >= 10
    hand = next(r for r in mlq if r["case"] == "hand-trace")
    assert hand["admitted_need"] == [30, 30, 30, 40, 50, 30]
    assert [a[0] for a in hand["admitted"]] == [0, 1, 2, 4, 5, 3]
    assert hand["consumed"] == [120, 40, 50] and hand["leftover"] == 30 and hand["stranded"] == [10, 0, 50]
    for res in mlq:
        assert sum(res["consumed"]) + res["leftover"] + sum(res["stranded"]) == sum(res["budgets"])
        admitted = [_req(aid, n) for _rid, aid, n in res["admitted"]]
        slots, ranks, ntok = batch_arrays(admitted, lambda a: int(a.split("-")[1]), rank_of_id)
        perm, off, sl, rk = build_segments_ref(slots, ranks, ntok)
        # stable group-by-slot keeps the admission order inside every segment
        tok_start = np.concatenate([[0], np.cumsum(ntok)])
        for s in range(len(sl)):
            reqs = [i for i in range(len(slots)) if slots[i] == sl[s]]
            want = np.concatenate([np.arange(tok_start[i], tok_start[i + 1]) for i in reqs]) if reqs else []
            assert perm[off[s]:off[s + 1]].tolist() == list(want)
