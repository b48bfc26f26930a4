"""Workload generators vs draws frozen from the reference
(tests/golden/workload_draws.json, oracle/gen_golden.py), plus BASELINE.json's C2 figures."""
import json

import numpy as np
import pytest

from paper_2411_17741_b200.model import build_catalog, zipf_catalog
from paper_2411_17741_b200.workload import (decode_batch, prefill_batch, rank_of_id, rank_probabilities,
                                            zipf_batch)


@pytest.fixture(scope="module")
def draws(golden_dir):
    return json.loads((golden_dir / "workload_draws.json").read_text())


def test_catalog_ids_match_reference(draws):
    assert list(build_catalog(100)) == draws["catalog_ids"]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_decode_batch_matches_reference_draws(draws, seed):
    assert decode_batch(seed) == draws["decode"][str(seed)]


@pytest.mark.parametrize("seed", [0, 1])
def test_zipf_batch_matches_reference_convention(draws, seed):
    assert zipf_batch(seed) == draws["zipf"][str(seed)]


def test_rank_probabilities_s1():
    p = rank_probabilities()
    assert p == pytest.approx([0.438, 0.219, 0.146, 0.1095, 0.0876], abs=5e-4)
    assert sum(p) == pytest.approx(1.0)


def test_c2_seed0_known_answers():
    """seed 0 -> 82 distinct adapters, sum of distinct ranks 3,808,
    sum rank x tokens 8,872 (the reference's adapter_units for this step)."""
    ids = decode_batch(0)
    distinct = set(ids)
    assert len(distinct) == 82
    assert sum(rank_of_id(a) for a in distinct) == 3808
    assert sum(rank_of_id(a) for a in ids) == 8872


def test_c3_prefill_rank_sum():
    ids, ntok = prefill_batch(0)
    assert len(ids) == 64 and ntok == [64] * 64
    assert sum(rank_of_id(a) for a in ids) == 1864


def test_zipf_catalog_convention():
    ids, probs = zipf_catalog(1000)
    assert ids[:6] == ["r8-0", "r16-0", "r32-0", "r64-0", "r128-0", "r8-1"]
    assert len(set(ids)) == 1000 and sum(probs) == pytest.approx(1.0)
    assert probs[0] / probs[1] == pytest.approx(2 ** 0.7)


@pytest.mark.reference
def test_live_assign_adapter_against_reference(reference_pkg):
    from adaptersim import model as rmodel
    from adaptersim import workload as rwl

    cfg = rmodel.WorkloadConfig(num_adapters=100)
    cat = rwl.build_catalog(cfg, rmodel.HardwareProfile())
    for seed in range(5, 12):
        rng = np.random.default_rng(seed)
        assert decode_batch(seed, 64) == [rwl.assign_adapter(rng, cfg, cat) for _ in range(64)]
