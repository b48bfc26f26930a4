"""Small decode + prefill applies for compute-sanitizer runs (memcheck / racecheck / synccheck).
Checks the result against the oracle as well."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.lora_ref import bf16_round, lora_apply_ref, make_adapters  # noqa: E402
from paper_2411_17741_b200.ops import build_segments, lora_apply_multi  # noqa: E402
from paper_2411_17741_b200.pool import AdapterPool  # noqa: E402


def main():
    rng = np.random.default_rng(3)
    h = 1024
    slot_ranks = {0: 8, 1: 24, 2: 64, 3: 128}
    adapters = [make_adapters(rng, slot_ranks, h, h, bf16=True) for _ in range(3)]
    npages = sum(-(-r // 8) for r in slot_ranks.values())
    pool = AdapterPool(npages, 1, [h] * 3, [h] * 3, dtype=torch.bfloat16, n_slots=4, max_tokens=512)
    page = 0
    for s, r in slot_ranks.items():
        n = -(-r // 8)
        pool.set_slot(s, r, list(range(page, page + n)))
        page += n
        pool.fill_async(s, pool.pack_host([torch.from_numpy(adapters[p][s][0]) for p in range(3)],
                                          [torch.from_numpy(adapters[p][s][1]) for p in range(3)], r))
    torch.cuda.synchronize()
    slots = [0, 1, 2, 3, 1, 0, 3, 2]
    ntok = [1, 2, 70, 3, 1, 65, 1, 2]  # decode segments and two prefill-routed ones
    tbl = build_segments(slots, [slot_ranks[s] for s in slots], ntok)
    T = sum(ntok)
    x = bf16_round(rng.standard_normal((T, h)).astype(np.float32))
    y0 = [bf16_round(rng.standard_normal((T, h)).astype(np.float32)) for _ in range(3)]
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    ys = [torch.from_numpy(y).cuda().to(torch.bfloat16) for y in y0]
    for _ in range(2):
        ys = [torch.from_numpy(y).cuda().to(torch.bfloat16) for y in y0]
        lora_apply_multi([xd] * 3, ys, tbl, pool=pool, layer=0, projs=[0, 1, 2])
    torch.cuda.synchronize()
    perm, off, sl, rk = tbl.to_host()
    for p in range(3):
        ref = bf16_round(lora_apply_ref(x, y0[p], perm, off, sl, rk, adapters[p]).astype(np.float32))
        np.testing.assert_allclose(ys[p].float().cpu().numpy(), ref, rtol=2e-2, atol=2e-2)
    pool.close()
    print("sanitize_small: decode + prefill applies match the oracle")


if __name__ == "__main__":
    main()
