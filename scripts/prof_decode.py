"""C2 decode applies for ncu captures: 4 layers x (q/k/v, o), eager, PDL-chained.
e.g. ncu --set full --import-source on -k regex:lora_apply_kernel -s 5 -c 2 -o OUT python scripts/prof_decode.py"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))
from paper_2411_17741_b200.executor import LoraStepExecutor  # noqa: E402
from trace_decode import H, P, setup  # noqa: E402


def main():
    NL = 4
    pool, req_slot, req_rank = setup()
    ex = LoraStepExecutor(pool, max_requests=1024, max_tokens=4096, proj_groups=[[0, 1, 2], [3]])
    T = len(req_slot)
    ex.upload(req_slot, req_rank, [1] * T)
    xs = [[torch.randn(T, H, device="cuda").to(torch.bfloat16) for _ in range(2)] for _ in range(NL)]
    ys = [[torch.randn(T, H, device="cuda").to(torch.bfloat16) for _ in range(P)] for _ in range(NL)]
    ex.build()
    for layer in range(NL):
        ex.apply_layer(layer, xs[layer], ys[layer], last=layer + 1 == NL)
    torch.cuda.synchronize()
    print("prof_decode: done")


if __name__ == "__main__":
    main()
