"""Per-item timeline of the decode kernel on the C2 workload (debug tool, run on the GPU box).

Prints, per launch: items per CTA, producer issue-to-consumer-start latency (load latency
as seen by the consumer), consumer busy time per item, producer inter-issue gap, and the
kernel span.  Saves the raw trace to gpurun_out/trace_<mode>.npy.
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
from paper_2411_17741_b200.model import build_catalog  # noqa: E402
from paper_2411_17741_b200.pool import AdapterPool, pages_for_rank  # noqa: E402
from paper_2411_17741_b200.workload import decode_batch, rank_of_id  # noqa: E402

H, L, P = 4096, 32, 4


def setup(n_layers=L):
    dev = torch.device("cuda", 0)
    catalog = build_catalog(100)
    ids = list(catalog)
    slot_of = {a: i for i, a in enumerate(ids)}
    n_pages = sum(pages_for_rank(s.rank) for s in catalog.values())
    pool = AdapterPool(n_pages, n_layers, [H] * P, [H] * P, dtype=torch.bfloat16, n_slots=len(ids),
                       max_tokens=4096, device=dev)
    page = 0
    for a in ids:
        r = catalog[a].rank
        npg = pages_for_rank(r)
        pool.set_slot(slot_of[a], r, list(range(page, page + npg)))
        buf = (torch.randn(npg * pool.page_bytes // 2, device=dev) * 0.02).to(torch.bfloat16)
        pool.fill_from_device(slot_of[a], buf.view(torch.uint8))
        page += npg
    batch = decode_batch(0, int(os.environ.get("TRACE_T", "256")))
    req_slot = [slot_of[a] for a in batch]
    req_rank = [rank_of_id(a) for a in batch]
    return pool, req_slot, req_rank


def analyze(tr, name):
    tr = tr.astype(np.int64)
    n_cta, cap, _ = tr.shape
    valid = tr[:, :, 0] > 0
    t0 = tr[:, :, 0][valid].min()
    issue = np.where(valid, tr[:, :, 0] - t0, 0)
    start = np.where(valid, tr[:, :, 2] - t0, 0)
    end = np.where(valid, tr[:, :, 3] - t0, 0)
    kind = (tr[:, :, 1] >> 32)
    nbytes = tr[:, :, 1] & 0xffffffff
    lat = (start - issue)[valid]
    busy = (end - start)[valid]
    per_cta = valid.sum(1)
    span = end.max()
    print(f"== {name}: span {span/1e3:.1f} us, items/CTA min {per_cta.min()} max {per_cta.max()} mean {per_cta.mean():.1f}, "
          f"bytes {nbytes[valid].sum()/1e6:.1f} MB -> {nbytes[valid].sum()/span:.0f} GB/s")
    for k, kn in ((1, "shrink"), (2, "expand")):
        m = valid & (kind == k)
        if m.any():
            l = (start - issue)[m]
            b = (end - start)[m]
            print(f"  {kn}: n={m.sum()} issue->start us p50 {np.median(l)/1e3:.2f} p90 {np.percentile(l,90)/1e3:.2f}; "
                  f"consumer busy us p50 {np.median(b)/1e3:.2f} p90 {np.percentile(b,90)/1e3:.2f} max {b.max()/1e3:.2f}")
    gaps = np.diff(np.sort(issue, axis=1), axis=1)
    gaps = np.diff(issue, axis=1)[valid[:, 1:] & valid[:, :-1]]
    print(f"  producer inter-issue gap us p50 {np.median(gaps)/1e3:.2f} p90 {np.percentile(gaps,90)/1e3:.2f}")
    it = tr[:, :, 4] - t0
    rd = tr[:, :, 5] - t0
    pre = (rd - it)[valid]
    post = (issue - rd)[valid]
    print(f"  producer: iteration-start -> stage free us p50 {np.median(pre)/1e3:.2f} p90 {np.percentile(pre,90)/1e3:.2f}; "
          f"stage free -> copies issued us p50 {np.median(post)/1e3:.2f} p90 {np.percentile(post,90)/1e3:.2f}")
    m6 = valid & (tr[:, :, 6] > 0)
    if m6.any():
        print(f"  producer unit prologue: dispatch us p50 {np.median(tr[:, :, 6][m6])/1e3:.2f} p90 {np.percentile(tr[:, :, 6][m6], 90)/1e3:.2f}; "
              f"decode us p50 {np.median(tr[:, :, 7][m6])/1e3:.2f} p90 {np.percentile(tr[:, :, 7][m6], 90)/1e3:.2f}")
    prev_issue_to_it = (it[:, 1:] - issue[:, :-1])[valid[:, 1:] & valid[:, :-1]]
    print(f"  producer: previous issue -> next iteration start us p50 {np.median(prev_issue_to_it)/1e3:.2f}")
    last_end = np.array([end[c, :per_cta[c]].max() if per_cta[c] else 0 for c in range(n_cta)])
    first_issue = np.array([issue[c, 0] for c in range(n_cta)])
    print(f"  CTA first-issue us p50 {np.median(first_issue)/1e3:.2f} max {first_issue.max()/1e3:.2f}; "
          f"CTA finish us min {last_end.min()/1e3:.1f} p50 {np.median(last_end)/1e3:.1f} max {last_end.max()/1e3:.1f}")


def main():
    pool, req_slot, req_rank = setup()
    ex = LoraStepExecutor(pool, max_requests=1024, max_tokens=4096, proj_groups=[[0, 1, 2], [3]])
    T = len(req_slot)
    ex.upload(req_slot, req_rank, [1] * T)
    xs = [torch.randn(T, H, device="cuda").to(torch.bfloat16) for _ in range(2)]
    ys = [torch.randn(T, H, device="cuda").to(torch.bfloat16) for _ in range(P)]
    ex.build()
    for _ in range(3):
        ex.apply_layer(5, xs, ys)
    torch.cuda.synchronize()
    cap = 512
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros(2, sm, cap, 8, dtype=torch.int64, device="cuda")
    _lib.call("cham_debug_set_trace", pool.handle, buf.data_ptr(), cap)
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    for name, projs in (("qkv", [0, 1, 2]), ("o", [3])):
        buf.zero_()
        from paper_2411_17741_b200.ops import lora_apply_multi, lora_apply_table
        if len(projs) > 1:
            lora_apply_multi([xs[0]] * 3, [ys[p] for p in projs], ex.table, pool=pool, layer=7, projs=projs)
        else:
            lora_apply_table(xs[1], ys[3], ex.table, pool=pool, layer=7, proj=3)
        torch.cuda.synchronize()
        tr = buf.cpu().numpy()[0]
        np.save(out / f"trace_{name}{os.environ.get('TRACE_TAG', '')}.npy", tr)
        analyze(tr, f"{name} fused kernel")
        valid = tr[:, :, 0] > 0
        t0 = tr[:, :, 0][valid].min()
        kind = tr[:, :, 1] >> 32
        for k, kn in ((1, "shrink"), (2, "expand")):
            m = valid & (kind == k)
            if m.any():
                print(f"   {kn} phase: first issue {(tr[:, :, 0][m].min() - t0) / 1e3:.1f} us, last consumer end "
                      f"{(tr[:, :, 3][m].max() - t0) / 1e3:.1f} us")
    _lib.call("cham_debug_set_trace", pool.handle, None, 0)


if __name__ == "__main__":
    main()
