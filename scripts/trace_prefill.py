"""Per-unit timeline of the fused tcgen05 prefill kernel on the C3 workload (debug tool, GPU box).

Per launch (q/k/v fused, then o): per unit kind the loader issue span, MMA span and epilogue
span, the epilogue lag behind the loader, and per-CTA start/finish spread.  Saves the raw
trace to gpurun_out/trace_prefill_<name>.npy.
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
from paper_2411_17741_b200.pool import AdapterPool, pages_for_rank  # noqa: E402
from paper_2411_17741_b200.workload import prefill_batch, rank_of_id  # noqa: E402

H, L, P = 4096, 2, 4


def main():
    dev = torch.device("cuda", 0)
    pids, pntok = prefill_batch(0)
    nseg = int(os.environ.get("TRACE_NSEG", "64"))
    pids, pntok = pids[:nseg], pntok[:nseg]
    ids = list(dict.fromkeys(pids))
    rank_of = {a: rank_of_id(a) for a in ids}
    slot_of = {a: i for i, a in enumerate(ids)}
    n_pages = sum(pages_for_rank(rank_of[a]) for a in ids)
    pool = AdapterPool(n_pages, L, [H] * P, [H] * P, dtype=torch.bfloat16, n_slots=len(ids), max_tokens=4096,
                       device=dev)
    page = 0
    for a in ids:
        npg = pages_for_rank(rank_of[a])
        pool.set_slot(slot_of[a], rank_of[a], list(range(page, page + npg)))
        buf = (torch.randn(npg * pool.page_bytes // 2, device=dev) * 0.02).to(torch.bfloat16)
        pool.fill_from_device(slot_of[a], buf.view(torch.uint8))
        page += npg
    ex = LoraStepExecutor(pool, max_requests=1024, max_tokens=4096, proj_groups=[[0, 1, 2], [3]])
    T = int(sum(pntok))
    ex.upload([slot_of[a] for a in pids], [rank_of[a] for a in pids], pntok)
    xs = [torch.randn(T, H, device=dev).to(torch.bfloat16) for _ in range(2)]
    ys = [torch.randn(T, H, device=dev).to(torch.bfloat16) for _ in range(P)]
    ex.build()
    for _ in range(3):
        ex.apply_layer(0, xs, ys)
    torch.cuda.synchronize()
    cap = 256
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros(2, sm, cap, 8, dtype=torch.int64, device=dev)
    _lib.call("cham_debug_set_trace", pool.handle, buf.data_ptr(), cap)
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    from paper_2411_17741_b200.ops import lora_apply_multi, lora_apply_table
    for name, projs in (("qkv", [0, 1, 2]), ("o", [3])):
        buf.zero_()
        if len(projs) > 1:
            lora_apply_multi([xs[0]] * 3, [ys[p] for p in projs], ex.table, pool=pool, layer=1, projs=projs)
        else:
            lora_apply_table(xs[1], ys[3], ex.table, pool=pool, layer=1, proj=3)
        torch.cuda.synchronize()
        tr = buf.cpu().numpy()[1].astype(np.int64)
        te = buf.cpu().numpy()[0].astype(np.int64)
        np.save(out / f"trace_prefill_epi_{name}.npy", te)
        np.save(out / f"trace_prefill_{name}.npy", tr)
        valid = tr[:, :, 0] > 0
        t0 = tr[:, :, 0][valid].min()
        T = np.where(tr > 0, tr - t0, 0) / 1e3
        kind = tr[:, :, 6] >> 32
        n = valid.sum(1)
        span = T[:, :, 5][valid].max()
        print(f"== {name}: span {span:.1f} us, units/CTA min {n.min()} max {n.max()} mean {n.mean():.1f}")

        def pct(a):
            return "p50 %.2f p90 %.2f" % (np.median(a), np.percentile(a, 90)) if len(a) else "-"
        for k, kn in ((1, "shrink"), (2, "expand"), (3, "vbuild")):
            m = valid & (kind == k)
            if not m.any():
                continue
            ok = m & (tr[:, :, 7] > 0) & (tr[:, :, 1] > 0)
            print(f"  {kn}: n={m.sum()}  first claim {T[:, :, 0][m].min():.1f} us, last claim {T[:, :, 0][m].max():.1f} us")
            print(f"    loader: claim->first slot {pct((T[:, :, 7] - T[:, :, 0])[ok])}; first slot->all issued {pct((T[:, :, 1] - T[:, :, 7])[ok])}")
            ok2 = m & (tr[:, :, 2] > 0) & (tr[:, :, 3] > 0) & (tr[:, :, 7] > 0)
            print(f"    MMA: slot->first stage full {pct((T[:, :, 2] - T[:, :, 7])[ok2])}; first full->last MMA issued {pct((T[:, :, 3] - T[:, :, 2])[ok2])}")
            ok3 = m & (tr[:, :, 4] > 0) & (tr[:, :, 5] > 0)
            print(f"    epilogue: acc ready->end {pct((T[:, :, 5] - T[:, :, 4])[ok3])}")
        E = np.where(te > 0, te - t0, 0) / 1e3
        me = (kind == 1) & (te[:, :, 0] > 0) & (te[:, :, 3] > 0)
        if me.any():
            print(f"    shrink epi detail: acc->drained {pct((E[:, :, 0] - T[:, :, 4])[me])}; drained->bar1 {pct((E[:, :, 1] - E[:, :, 0])[me])}; "
                  f"bar1->atomic {pct((E[:, :, 2] - E[:, :, 1])[me])}; atomic->bar2 {pct((E[:, :, 3] - E[:, :, 2])[me])}")
        ml = me & (te[:, :, 5] > 0)
        if ml.any():
            print(f"    last-arriver: bar2->reduced {pct((E[:, :, 4] - E[:, :, 3])[ml])}; reduced->published {pct((E[:, :, 5] - E[:, :, 4])[ml])}")
        fin = np.array([T[c, :n[c], 5].max() if n[c] else 0 for c in range(sm)])
        print(f"  CTA finish us min {fin.min():.1f} p50 {np.median(fin):.1f} max {fin.max():.1f}")
    _lib.call("cham_debug_set_trace", pool.handle, None, 0)


if __name__ == "__main__":
    main()
