"""Self-checks of the CPU oracle (oracle/), which the GPU parity tests trust.

LoRA numeric parity is unpinned by the reference: these tests pin the oracle to
its definition y += (x.A).B instead — an independent dense formulation, linearity,
shrink∘expand == apply, bf16 rounding against torch — and to SURVEY §8d's C1/C2 figures.
"""
import numpy as np
import pytest
import torch

from oracle.lora_ref import (algorithmic_bytes, bf16_bits, bf16_from_bits, bf16_round, lora_apply_ref,
                             lora_expand_ref, lora_shrink_ref, make_adapters)
from oracle.segments_ref import build_segments_ref
from paper_2411_17741_b200.workload import decode_batch, rank_of_id


def _c1(seed=0):
    """h=4096, ranks [8, 8, 16, 16], 32 decode tokens,
    request -> adapter from default_rng(0).integers(0, 4, 32)."""
    rng = np.random.default_rng(seed)
    req_slot = np.random.default_rng(0).integers(0, 4, 32).astype(np.int32)
    ranks = {0: 8, 1: 8, 2: 16, 3: 16}
    adapters = make_adapters(rng, ranks, 4096, 4096)
    x = rng.standard_normal((32, 4096)).astype(np.float32)
    y = rng.standard_normal((32, 4096)).astype(np.float32)
    req_rank = np.array([ranks[s] for s in req_slot], dtype=np.int32)
    return x, y, adapters, req_slot, req_rank, np.ones(32, np.int32)


def test_apply_matches_dense_per_token_definition():
    x, y, adapters, req_slot, req_rank, ntok = _c1()
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(req_slot, req_rank, ntok)
    got = lora_apply_ref(x, y, perm, seg_off, seg_slot, seg_rank, adapters)
    want = y.astype(np.float64).copy()
    for t in range(32):
        a, b = adapters[int(req_slot[t])]
        want[t] += (x[t].astype(np.float64) @ a.astype(np.float64)) @ b.astype(np.float64)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def test_apply_linearity_and_perm_invariance():
    x, y, adapters, req_slot, req_rank, ntok = _c1(1)
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(req_slot, req_rank, ntok)
    z = np.zeros_like(y)
    d1 = lora_apply_ref(x, z, perm, seg_off, seg_slot, seg_rank, adapters)
    d2 = lora_apply_ref(2.5 * x.astype(np.float64), z, perm, seg_off, seg_slot, seg_rank, adapters)
    np.testing.assert_allclose(d2, 2.5 * d1, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(lora_apply_ref(x, y, perm, seg_off, seg_slot, seg_rank, adapters), y + d1,
                               rtol=1e-12, atol=1e-12)


def test_shrink_then_expand_equals_apply():
    x, y, adapters, req_slot, req_rank, ntok = _c1(2)
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(req_slot, req_rank, ntok)
    v = lora_shrink_ref(x, perm, seg_off, seg_slot, seg_rank, adapters, 16)
    assert v.shape == (32, 16)
    got = lora_expand_ref(v, y, perm, seg_off, seg_slot, seg_rank, adapters)
    np.testing.assert_allclose(got, lora_apply_ref(x, y, perm, seg_off, seg_slot, seg_rank, adapters),
                               rtol=1e-12, atol=1e-12)


def test_no_adapter_segments_leave_y():
    rng = np.random.default_rng(3)
    adapters = make_adapters(rng, {0: 8}, 64, 64)
    x = rng.standard_normal((4, 64)).astype(np.float32)
    y = rng.standard_normal((4, 64)).astype(np.float32)
    perm, seg_off, seg_slot, seg_rank = build_segments_ref([-1, 0, -1, 0], [0, 8, 0, 8], [1, 1, 1, 1])
    out = lora_apply_ref(x, y, perm, seg_off, seg_slot, seg_rank, adapters)
    np.testing.assert_array_equal(out[[0, 2]], y[[0, 2]])
    assert not np.allclose(out[[1, 3]], y[[1, 3]])


def test_bf16_rounding_matches_torch():
    rng = np.random.default_rng(4)
    a = np.concatenate([rng.standard_normal(10000).astype(np.float32) * 10.0 ** rng.integers(-30, 30, 10000),
                        np.array([0.0, -0.0, np.inf, -np.inf, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8], np.float32)])
    want = torch.from_numpy(a).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(bf16_round(a), want)
    np.testing.assert_array_equal(bf16_from_bits(bf16_bits(a)), want)
    assert np.isnan(bf16_round(np.array([np.nan], np.float32)))[0]


def test_c2_algorithmic_bytes():
    """SURVEY §8d C2 seed 0: 7.99 GB of adapter bytes + 0.81 GB of activations per step."""
    ids = decode_batch(0)
    slot = {a: i for i, a in enumerate(sorted(set(ids)))}
    perm, seg_off, seg_slot, seg_rank = build_segments_ref([slot[a] for a in ids], [rank_of_id(a) for a in ids],
                                                           [1] * 256)
    ad, act = algorithmic_bytes(seg_off, seg_slot, seg_rank, 256, 4096, 4096, 2, 2, 2)
    assert ad * 128 == 3808 * 8192 * 2 * 128
    assert ad * 128 / 1e9 == pytest.approx(7.99, abs=0.005)
    assert act * 128 / 1e9 == pytest.approx(0.81, abs=0.005)
