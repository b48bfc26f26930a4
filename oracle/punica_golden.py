"""Third-party golden vectors for the LoRA apply (test infrastructure only).

The reference (adaptersim) never computes y += (x.A_i).B_i: PAPER.md:139-141 delegates the
kernels to S-LoRA, which is not vendored and has no pinned version in any manifest.  The
published algorithm S-LoRA's kernels implement is Punica's SGMV (segmented gather
matrix-vector): per segment s of consecutive (grouped) tokens with LoRA index l_s,
    shrink:  v[t, :]  = scaling * x[t, :] @ A_{l_s}^T        A stacked [n_lora, max_rank, h_in]
    expand:  y[t, :] += v[t, :] @ B_{l_s}^T                  B stacked [n_lora, h_out, max_rank]
Heterogeneous ranks are the zero-padded rows/columns beyond r_i (S-LoRA's unified paging
stores rank-r_i tiles; the padding contributes exact zeros).

The pinned third-party implementation used here is vLLM 0.22.0's torch restatement of the
Punica ops, `vllm/lora/ops/torch_ops/lora_ops.py` (`sgmv_shrink`, `sgmv_expand`, both
expanding seq_len_tensor into per-token LoRA indices and doing one einsum), installed in this
image.  `main()` (run in this container: `python -m oracle.punica_golden`) evaluates it in fp32
on CPU over seeded inputs and commits `tests/golden/punica_sgmv.npz`; the inputs are
regenerated from the seed by `case_inputs` (their SHA-256 is stored so a drift of the RNG
stream fails loudly instead of silently comparing different data).  The tests pin
`oracle/lora_ref.py` to these outputs (CPU) and check the CUDA path against them (GPU).

Batch construction follows the reference: per-request (slot, rank, tokens) in batch order
(engine.py:64-76), grouped by slot with the stable segment builder (oracle/segments_ref.py).
"""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

from oracle.lora_ref import bf16_round, make_adapters
from oracle.segments_ref import build_segments_ref

GOLDEN = Path(__file__).resolve().parents[1] / "tests" / "golden" / "punica_sgmv.npz"

# name -> (seed, h_in, h_out, slot ranks, request slots, request tokens, bf16-rounded inputs)
CASES = {
    # SURVEY §8(d) C1 / BASELINE configs[0]: h=4096, 32 decode requests over 4 adapters of
    # ranks {8, 16}, fp32 (slots = default_rng(0).integers(0, 4, 32), as tests/test_lora_gpu.py)
    "c1_fp32": (0, 4096, 4096, {0: 8, 1: 8, 2: 16, 3: 16},
                np.random.default_rng(0).integers(0, 4, 32).tolist(), [1] * 32, False),
    # mixed ranks 8..128 (+ ranks that are not multiples of 8), fp32, multi-token segments
    "mixed_fp32": (11, 1024, 1024, {0: 8, 1: 24, 2: 40, 3: 128, 5: 64},
                   [3, 0, 5, 1, 2, 3, 0, 5, 2, 1, 3, 3, 0, 2, 5, 1, 0, 2, 3, 5],
                   [1, 2, 1, 4, 1, 3, 1, 2, 1, 1, 2, 1, 1, 4, 1, 1, 3, 1, 1, 2], False),
    # bf16-rounded inputs, decode tokens, ranks 8..128, rectangular (h_out < h_in)
    "decode_bf16": (12, 2048, 1024, {0: 8, 1: 16, 2: 32, 3: 64, 4: 128},
                    np.random.default_rng(12).integers(0, 5, 48).tolist(), [1] * 48, True),
    # bf16-rounded inputs, prefill-sized segments (>= 64 tokens take the tcgen05 route on a
    # bf16 pool) mixed with decode tokens
    "prefill_bf16": (13, 2048, 512, {0: 16, 1: 64, 2: 128, 3: 8},
                     [2, 0, 1, 3, 2, 0, 1], [64, 5, 80, 1, 3, 2, 1], True),
}


def case_inputs(name: str):
    """Regenerate a case's inputs: (adapters slot -> (A [h_in, r], B [r, h_out]), x, y0,
    perm, seg_off, seg_slot, seg_rank), in the order tests/test_lora_gpu.py:_run_case uses."""
    seed, h_in, h_out, slot_ranks, slots, ntok, bf16 = CASES[name]
    rng = np.random.default_rng(seed)
    adapters = make_adapters(rng, slot_ranks, h_in, h_out, bf16=bf16)
    T = int(np.sum(ntok))
    x = rng.standard_normal((T, h_in)).astype(np.float32)
    y0 = rng.standard_normal((T, h_out)).astype(np.float32)
    if bf16:
        x, y0 = bf16_round(x), bf16_round(y0)
    ranks = [slot_ranks[s] for s in slots]
    perm, seg_off, seg_slot, seg_rank = build_segments_ref(slots, ranks, ntok)
    return adapters, x, y0, perm, seg_off, seg_slot, seg_rank


def inputs_sha(adapters, x, y0) -> str:
    h = hashlib.sha256()
    for s in sorted(adapters):
        h.update(np.ascontiguousarray(adapters[s][0]).tobytes())
        h.update(np.ascontiguousarray(adapters[s][1]).tobytes())
    h.update(x.tobytes())
    h.update(y0.tobytes())
    return h.hexdigest()


def punica_apply(name: str) -> np.ndarray:
    """y0 + LoRA(x) through vLLM's Punica torch ops (fp32, CPU)."""
    import torch
    from vllm.lora.ops.torch_ops.lora_ops import sgmv_expand, sgmv_shrink

    adapters, x, y0, perm, seg_off, seg_slot, seg_rank = case_inputs(name)
    slots = sorted(adapters)
    max_r = max(adapters[s][0].shape[1] for s in slots)
    h_in, h_out = x.shape[1], y0.shape[1]
    lora_a = torch.zeros(len(slots), max_r, h_in)
    lora_b = torch.zeros(len(slots), h_out, max_r)
    for i, s in enumerate(slots):
        a, b = adapters[s]
        lora_a[i, : a.shape[1]] = torch.from_numpy(a.T.copy())
        lora_b[i, :, : b.shape[0]] = torch.from_numpy(b.T.copy())
    perm_t = torch.as_tensor(np.asarray(perm, dtype=np.int64))
    lens = torch.as_tensor(np.diff(np.asarray(seg_off, dtype=np.int64)))
    starts = torch.as_tensor(np.asarray(seg_off[:-1], dtype=np.int64))
    idx = torch.as_tensor([slots.index(int(s)) for s in seg_slot], dtype=torch.int64)
    n_tok = int(seg_off[-1])
    xs = torch.from_numpy(x)[perm_t]                      # grouped (gathered) token rows
    ys = torch.from_numpy(y0)[perm_t].clone()
    v = torch.zeros(n_tok, max_r)
    sgmv_shrink(xs, lora_a, v, starts, lens, idx, len(seg_slot), int(lens.max()), n_tok, 1.0)
    sgmv_expand(v, lora_b, ys, starts, lens, idx, len(seg_slot), int(lens.max()), n_tok, add_inputs=True)
    out = y0.copy()
    out[np.asarray(perm, dtype=np.int64)] = ys.numpy()
    return out


def main():
    import vllm

    arrays, meta = {}, {"generator": "vllm.lora.ops.torch_ops.lora_ops sgmv_shrink/sgmv_expand",
                        "vllm_version": vllm.__version__, "cases": {}}
    for name in CASES:
        adapters, x, y0, *_ = case_inputs(name)
        arrays[name] = punica_apply(name).astype(np.float32)
        meta["cases"][name] = {"inputs_sha256": inputs_sha(adapters, x, y0)}
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(GOLDEN, **arrays)
    print(f"wrote {GOLDEN} ({GOLDEN.stat().st_size} bytes): {sorted(CASES)}")


def load_golden():
    z = np.load(GOLDEN)
    meta = json.loads(bytes(z["meta"]).decode())
    return {k: z[k] for k in z.files if k != "meta"}, meta


if __name__ == "__main__":
    main()
