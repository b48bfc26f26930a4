"""Summarise an `ncu --set full` report: per launch duration, DRAM bytes, throughput, tensor
pipe, occupancy.  Writes profiles/traffic_<tag>.json (per-launch DRAM traffic that bench.py
reports as roofline.traffic) and prints a markdown table.

usage: python scripts/ncu_summary.py <report.ncu-rep> <tag>
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = {
    "gpu__time_duration.sum": "time_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard": "stall_long_sb",
}


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, rows = rows[0], rows[1], rows[2:]
    scale = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    launches = []
    for r in rows:
        d = {"kernel": r[hdr.index("Kernel Name")][:80]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    d[name] = float(r[i].replace(",", "")) * scale.get(units[i], 1)
                except ValueError:
                    pass
        launches.append(d)
    traffic = [l.get("dram_read", 0) + l.get("dram_write", 0) for l in launches]
    summary = {"report": Path(rep).name, "launches": launches,
               "traffic_per_launch": sum(traffic) / max(1, len(traffic))}
    (ROOT / "profiles" / f"traffic_{tag}.json").write_text(json.dumps(summary, indent=1))
    print(f"| launch | kernel | us | DRAM read MB | DRAM write MB | GB/s | L2 MB | tensor % | warps active % |")
    print("|---|---|---|---|---|---|---|---|---|")
    for i, l in enumerate(launches):
        t = l.get("time_ns", 0)
        rd, wr = l.get("dram_read", 0), l.get("dram_write", 0)
        print(f"| {i} | {l['kernel'][:40]} | {t / 1e3:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
              f"{(rd + wr) / max(t, 1):.0f} | {l.get('l2_bytes', 0) / 1e6:.1f} | {l.get('tensor_pct', 0):.1f} | "
              f"{l.get('warps_active_pct', 0):.1f} |")


if __name__ == "__main__":
    main()
