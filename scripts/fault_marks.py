"""Analyse gpurun_out/fault_trace_<i>.npy of a faulting run: the hung launch's incomplete units
and the MMA warp's last progress mark of every CTA (CHAM_PF_WATCHDOG trace builds)."""
import sys

import numpy as np

for i in sys.argv[1:]:
    tr = np.load(f"gpurun_out/fault_trace_{i}.npy")
    cap = tr.shape[1]
    cr = tr[:, cap - 1, :].copy()
    ep = cr[:, 6]
    old = ep.min()
    if (ep == old).all():
        print(i, "no hung launch")
        continue
    tw = cr[ep == old, 2].min()
    marks = tr[:, cap - 15, :]
    print(f"run {i}: hung launch {old}")
    for b in range(tr.shape[0]):
        for k in range(cap - 15):
            r = tr[b, k]
            if r[0] >= tw and r[0] > 0 and not r[5] >= tw:
                kind = int(r[6] >> 32)
                f3 = int(r[3])
                if f3 >> 62 == 1:
                    print(f"    in-unit MMA progress: stage {(f3 >> 8) & 0xffffff} state {f3 & 0xff} "
                          "(1 waiting for full, 2 issuing, 3 issued+committed)")
                m = marks[b]
                print(f"  cta {b} k {k} kind {kind} unit {int(r[6] & 0xffffffff)}; last MMA mark: ep {int(m[5])} "
                      f"unit k {int(m[0])} stage {int(m[1])} seq {int(m[2])} state {int(m[3])} "
                      f"t {(int(m[4]) - tw) / 1e3:.1f} us")
