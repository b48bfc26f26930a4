"""Aggregate an ncu --csv launch list (gpurun_out/launches_*.csv) per kernel name."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = collections.defaultdict(dict)
    names = {}
    for r in rows:
        d[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki][:70]
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for i, m in d.items():
        cnt[names[i]] += 1
        for k, v in m.items():
            agg[names[i]][k] += v
    print(f)
    for n, a in agg.items():
        c = cnt[n]
        t = a["gpu__time_duration.sum"]
        rd, wr = a["dram__bytes_read.sum"], a["dram__bytes_write.sum"]
        extra = ""
        if "lts__t_bytes.sum" in a:
            extra += f" L2MB={a['lts__t_bytes.sum'] / c / 1e6:8.1f}"
        k = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
        if k in a:
            extra += f" tensor%={a[k] / c:.1f}"
        print(f"  {n:70s} n={c:4d} avg_us={t / c / 1e3:8.2f} rdMB={rd / c / 1e6:8.1f} wrMB={wr / c / 1e6:7.1f} "
              f"GB/s={(rd + wr) / max(t, 1):7.0f}{extra}")
