"""GPU parity against third-party golden vectors (vLLM 0.22.0 Punica SGMV, fp32 on CPU; see
oracle/punica_golden.py): the CUDA path through the C ABI on the same inputs.  fp32 rtol 1e-5;
bf16 (inputs bf16-rounded, fp32 accumulate) rtol 2e-2 against the golden output rounded to
bf16 (north star).  Both routes: the default (segments >= 64 tokens of a bf16 pool on the
tcgen05 kernel) and decode-kernel only."""
import numpy as np
import pytest
import torch

from oracle.lora_ref import bf16_round
from oracle.punica_golden import CASES, case_inputs, load_golden

pytestmark = pytest.mark.gpu

GOLD, _ = load_golden()


@pytest.mark.parametrize("route", ["default", "decode_only"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_cuda_path_matches_punica_golden(name, route):
    from paper_2411_17741_b200.ops import lora_apply
    from paper_2411_17741_b200.pool import AdapterPool

    adapters, x, y0, perm, seg_off, seg_slot, seg_rank = case_inputs(name)
    bf16 = CASES[name][6]
    dtype = torch.bfloat16 if bf16 else torch.float32
    h_in, h_out = x.shape[1], y0.shape[1]
    npages = sum(-(-a.shape[1] // 8) for a, _ in adapters.values())
    pool = AdapterPool(npages, 1, [h_in], [h_out], dtype=dtype, n_slots=max(adapters) + 1, max_tokens=4096)
    if route == "decode_only":
        pool.set_prefill_route(0)
    page = 0
    for s, (a, b) in adapters.items():
        r = a.shape[1]
        npg = -(-r // 8)
        pool.set_slot(s, r, list(range(page, page + npg)))
        page += npg
        pool.fill_async(s, pool.pack_host([torch.from_numpy(a)], [torch.from_numpy(b)], r))
    torch.cuda.synchronize()
    xd = torch.from_numpy(x).to("cuda", dtype)
    yd = torch.from_numpy(y0).to("cuda", dtype)
    lora_apply(xd, yd, seg_slot, seg_off, seg_rank, pool=pool, layer=0, proj=0, perm=perm)
    torch.cuda.synchronize()
    pool.check_device_error()
    got = yd.float().cpu().numpy()
    pool.close()
    if bf16:
        np.testing.assert_allclose(got, bf16_round(GOLD[name]), rtol=2e-2, atol=2e-2)
    else:
        np.testing.assert_allclose(got, GOLD[name], rtol=1e-5, atol=1e-5)
