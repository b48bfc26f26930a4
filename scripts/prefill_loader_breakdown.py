"""Per-unit breakdown of the prefill loader loop (expand units of the q/k/v launch) from the
traces scripts/trace_prefill.py saves (gpurun_out/trace_prefill_{,epi_}qkv.npy); run here after
the GPU call.  Fields: see trace_ld / trace_put in cham_prefill.cu."""
import numpy as np
tr = np.load("gpurun_out/trace_prefill_qkv.npy").astype(np.int64)
te = np.load("gpurun_out/trace_prefill_epi_qkv.npy").astype(np.int64)
G, K, _ = tr.shape
kind = tr[:, :, 6] >> 32
rows = []
for c in range(G):
    for k in range(1, K - 1):
        if kind[c, k] != 2 or tr[c, k, 0] == 0 or tr[c, k, 1] == 0 or tr[c, k - 1, 1] == 0: continue
        top = tr[c, k - 1, 1]; nxt = tr[c, k, 1]
        e = te[c, k]
        if (e[[0, 1, 7, 2, 3, 4, 5]] == 0).any(): continue
        rows.append([e[0] - top, e[1] - e[0], e[7] - e[1], tr[c, k, 0] - e[7], e[2] - tr[c, k, 0], e[3] - e[2], e[4] - e[3], e[5] - e[4], nxt - e[5], nxt - top])
r = np.array(rows) / 1e3
names = ["publish(uempty)", "advance(claim)", "peek+prefetch", "make_unit", "vempty wait", "tile ready+fences", "V copy issue", "ring slot wait", "B copies..next top", "TOTAL"]
print("n", len(r))
for i, n in enumerate(names):
    print(f"{n:22s} p50 {np.percentile(r[:, i], 50):6.3f}  mean {r[:, i].mean():6.3f}  p90 {np.percentile(r[:, i], 90):6.3f}")
