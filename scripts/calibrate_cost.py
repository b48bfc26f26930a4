"""Calibrate the B200 LoRA latency model (paper_2411_17741_b200/cost_model.py) on the GPU box.

Measures one step's LoRA apply (32 layers x q/k/v/o at Llama-2-7B dims, CUDA-graph replay,
inputs resident in HBM) for decode batches of 8..256 tokens and prefill batches of 8..64
segments x 64 tokens, fits `t = base + c_gb * adapter_GB + c_tok * tokens` per path, and writes
profiles/lora_cost_b200.json (the table B200CostModel loads).
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2411_17741_b200.cost_model import Geometry, LoraLatencyModel  # noqa: E402
from paper_2411_17741_b200.executor import LoraStepExecutor  # noqa: E402
from paper_2411_17741_b200.model import build_catalog  # noqa: E402
from paper_2411_17741_b200.pool import AdapterPool, pages_for_rank  # noqa: E402
from paper_2411_17741_b200.workload import decode_batch, prefill_batch, rank_of_id  # noqa: E402

H, L, P = 4096, 32, 4


def main():
    dev = torch.device("cuda", 0)
    catalog = build_catalog(100)
    ids = list(catalog)
    for seed in range(3):
        for a in prefill_batch(seed)[0]:
            if a not in ids:
                ids.append(a)
    rank_of = {a: rank_of_id(a) for a in ids}
    slot_of = {a: i for i, a in enumerate(ids)}
    pool = AdapterPool(sum(pages_for_rank(rank_of[a]) for a in ids), L, [H] * P, [H] * P, dtype=torch.bfloat16,
                       n_slots=len(ids), max_tokens=4096, device=dev)
    page = 0
    for a in ids:
        n = pages_for_rank(rank_of[a])
        pool.set_slot(slot_of[a], rank_of[a], list(range(page, page + n)))
        buf = (torch.randn(n * pool.page_bytes // 2, device=dev) * 0.02).to(torch.bfloat16)
        pool.fill_from_device(slot_of[a], buf.view(torch.uint8))
        page += n
        del buf
    geom = Geometry()
    xs = [[torch.randn(4096, H, device=dev).to(torch.bfloat16) for _ in range(2)] for _ in range(L)]
    ys = [[torch.randn(4096, H, device=dev).to(torch.bfloat16) for _ in range(P)] for _ in range(L)]

    def measure(batch, ntok):
        ex = LoraStepExecutor(pool, max_requests=1024, max_tokens=4096, proj_groups=[[0, 1, 2], [3]])
        T = int(sum(ntok))
        ex.upload([slot_of[a] for a in batch], [rank_of[a] for a in batch], ntok)
        xv = [[x[:T] for x in layer] for layer in xs]
        yv = [[y[:T] for y in layer] for layer in ys]
        s = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(s):
            ex.run(xv, yv)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ex.run(xv, yv)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(10):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 10
        gb = sum(geom.adapter_bytes(rank_of[a]) for a in set(batch)) / 1e9
        return gb, T, us

    dec, pre = [], []
    for T in (8, 16, 32, 64, 128, 256):
        for seed in range(3):
            dec.append(measure(decode_batch(seed, T, 100), [1] * T))
            print("decode", T, seed, dec[-1], flush=True)
    for nseg in (8, 16, 32, 64):
        for seed in range(3):
            pids, pn = prefill_batch(seed)
            pre.append(measure(pids[:nseg], pn[:nseg]))
            print("prefill", nseg, seed, pre[-1], flush=True)
    model = LoraLatencyModel(LoraLatencyModel.fit_path(dec), LoraLatencyModel.fit_path(pre), geom,
                             source="scripts/calibrate_cost.py on 1x B200 (CUDA-graph step of 32 layers x q/k/v/o, "
                                    "bf16, inputs in HBM)")
    d = model.to_json()
    d["samples"] = {"decode": dec, "prefill": pre}
    for name, samples, coef in (("decode", dec, model.decode), ("prefill", pre, model.prefill)):
        err = [abs(coef(gb, t) - us) / us for gb, t, us in samples]
        d[f"{name}_max_rel_err"] = max(err)
        print(name, coef, "max rel err %.3f" % max(err))
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "lora_cost_b200.json").write_text(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
