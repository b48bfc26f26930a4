"""Timeline of a PDL-chained sequence of decode applies (C2 batch, debug tool, GPU box).

Launches layers 0..NL-1 x (q/k/v, o) eagerly on one stream, each apply with its own slice of
the debug trace buffer (cham_debug_set_trace before every launch), then prints per launch:
first copy issued, first consumer start, last consumer end (all relative to the first launch),
the gap to the previous launch's end, the CTA finish spread, and a bandwidth timeline
(bytes whose consumer finished in each 1 us bin).  Saves gpurun_out/trace_chain.npy.
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2411_17741_b200 import _lib  # noqa: E402
from paper_2411_17741_b200.executor import LoraStepExecutor  # noqa: E402

sys.path.insert(0, str(ROOT / "scripts"))
from trace_decode import H, P, setup  # noqa: E402


def main():
    NL = int(os.environ.get("TRACE_LAYERS", "4"))
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
    cap = 256
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    n_launch = 2 * NL
    buf = torch.zeros(n_launch, 2, sm, cap, 8, dtype=torch.int64, device="cuda")
    from paper_2411_17741_b200.ops import lora_apply_multi, lora_apply_table

    s = torch.cuda.current_stream()
    k = 0
    for layer in range(NL):
        for g, projs in enumerate(ex.proj_groups):
            _lib.call("cham_debug_set_trace", pool.handle, buf[k].data_ptr(), cap)
            if ex.l2_prefetch_bytes > 0:
                if g + 1 < len(ex.proj_groups):
                    pool.set_next_apply(layer, ex.proj_groups[g + 1])
                elif layer + 1 < NL:
                    pool.set_next_apply(layer + 1, ex.proj_groups[0])
            if len(projs) > 1:
                lora_apply_multi([xs[layer][g]] * len(projs), [ys[layer][p] for p in projs], ex.table, pool=pool,
                                 layer=layer, projs=projs)
            else:
                lora_apply_table(xs[layer][g], ys[layer][projs[0]], ex.table, pool=pool, layer=layer, proj=projs[0])
            k += 1
    torch.cuda.synchronize()
    _lib.call("cham_debug_set_trace", pool.handle, None, 0)
    tr = buf.cpu().numpy()[:, 0].astype(np.int64)  # [launch][cta][seq][8]
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    np.save(out / f"trace_chain{os.environ.get('TRACE_TAG', '')}.npy", tr)
    life = tr[:, :, cap - 1, :].copy()  # per-CTA stamps: entry, plan ready, -, consumers done, exit
    tr = tr[:, :, :cap - 1]
    valid = tr[..., 0] > 0
    t0 = tr[..., 0][valid].min()
    prev_end = None
    tot_bytes = 0
    print(f"chain of {n_launch} applies (layers 0..{NL - 1} x q/k/v + o), C2 batch, {T} tokens")
    for i in range(n_launch):
        v = valid[i]
        issue = tr[i, :, :, 0] - t0
        start = tr[i, :, :, 2] - t0
        end = tr[i, :, :, 3] - t0
        nb = (tr[i, :, :, 1] & 0xffffffff)
        first_issue = issue[v].min()
        first_start = start[v].min()
        last_end = end[v].max()
        cta_end = np.array([end[c][v[c]].max() if v[c].any() else 0 for c in range(v.shape[0])])
        cta_first = np.array([issue[c][v[c]].min() if v[c].any() else 0 for c in range(v.shape[0])])
        b = nb[v].sum()
        tot_bytes += b
        gap = "" if prev_end is None else f" gap-from-prev-end {(first_issue - prev_end) / 1e3:+.2f}"
        print(f"[{i}] {'qkv' if i % 2 == 0 else 'o  '} issue {first_issue / 1e3:7.2f} start {first_start / 1e3:7.2f} "
              f"end {last_end / 1e3:7.2f} span {(last_end - first_issue) / 1e3:5.2f} us{gap}; "
              f"CTA first-issue p50 {np.median(cta_first) / 1e3 - first_issue / 1e3:.2f} max "
              f"{(cta_first.max() - first_issue) / 1e3:.2f}; CTA end min {cta_end.min() / 1e3:.2f} p10 "
              f"{np.percentile(cta_end, 10) / 1e3:.2f} p50 {np.median(cta_end) / 1e3:.2f}; "
              f"{b / 1e6:.1f} MB -> {b / max(1, last_end - first_issue):.0f} GB/s")
        ent, pln, dn, ex_ = (life[i, :, j] - t0 for j in (0, 1, 3, 4))
        print(f"     CTA entry min {ent.min() / 1e3:7.2f} p50 {np.median(ent) / 1e3:7.2f} max {ent.max() / 1e3:7.2f}; "
              f"plan-ready - entry p50 {np.median(pln - ent) / 1e3:.2f}; exit - consumers-done p50 "
              f"{np.median(ex_ - dn) / 1e3:.2f} max {(ex_ - dn).max() / 1e3:.2f}; exit min {ex_.min() / 1e3:7.2f} "
              f"max {ex_.max() / 1e3:7.2f}")
        prev_end = last_end
    span = max(tr[i, :, :, 3][valid[i]].max() for i in range(n_launch)) - t0
    print(f"total {tot_bytes / 1e6:.1f} MB in {span / 1e3:.1f} us -> {tot_bytes / span:.0f} GB/s")
    # bandwidth timeline: bytes of items whose consumer ended in each 1 us bin
    ends = (tr[..., 3] - t0)[valid]
    bytes_ = (tr[..., 1] & 0xffffffff)[valid]
    bins = np.zeros(int(span // 1000) + 1)
    np.add.at(bins, (ends // 1000).astype(np.int64), bytes_)
    line = " ".join(f"{x / 1e6:.1f}" for x in bins)  # bytes per us / 1e6 = TB/s
    print("GB/s per 1us bin (TB/s):", line)


if __name__ == "__main__":
    main()
