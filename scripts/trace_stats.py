"""Summaries of gpurun_out/trace_<name>.npy (written by scripts/trace_decode.py)."""
import sys
import numpy as np

for name in sys.argv[1:] or ["qkv", "o"]:
    tr = np.load(f"gpurun_out/trace_{name}.npy").astype(np.int64)
    valid = tr[:, :, 0] > 0
    t0 = tr[:, :, 0][valid].min()
    issue = tr[:, :, 0] - t0; it = tr[:, :, 4] - t0; rd = tr[:, :, 5] - t0
    kind = tr[:, :, 1] >> 32; start = tr[:, :, 2] - t0; end = tr[:, :, 3] - t0; nb = tr[:, :, 1] & 0xffffffff
    n = valid.sum(1)
    for kk, nm0 in ((1, "shrink"), (2, "expand")):
        pg, cb, busy, iss, per = [], [], [], [], []
        for c in range(tr.shape[0]):
            ks = [k for k in range(n[c]) if kind[c, k] == kk]
            for k in ks[1:]:
                pg.append(it[c, k] - issue[c, k - 1]); cb.append(start[c, k] - end[c, k - 1])
                busy.append(end[c, k] - start[c, k]); iss.append(issue[c, k] - rd[c, k])
            if len(ks) > 3:
                per.append((end[c, ks[-1]] - start[c, ks[0]]) / len(ks))
        for nm, a in (("producer gap", pg), ("producer issue", iss), ("consumer idle", cb), ("consumer busy", busy),
                      ("CTA stage period", per)):
            a = np.array(a) / 1e3
            print(f"{name:4s} {nm0:7s} {nm:17s} p10/50/75/90", np.percentile(a, [10, 50, 75, 90]).round(2))
        m = valid & (kind == kk)
        st = np.array([start[c][m[c]].min() for c in range(len(n)) if m[c].any()]) / 1e3
        fin = np.array([end[c][m[c]].max() for c in range(len(n)) if m[c].any()]) / 1e3
        print(f"{name:4s} {nm0:7s} CTA start min/p50/max", np.percentile(st, [0, 50, 100]).round(1),
              " finish", np.percentile(fin, [0, 50, 100]).round(1), f" bytes {nb[m].sum()/1e6:.1f} MB")
