#!/usr/bin/env python
"""Benchmark: batched heterogeneous-rank LoRA apply on B200 (BASELINE.json metric).

Workload (N=1 line): BASELINE config C2 — Llama-2-7B dims (h=4096, 32 layers, q/k/v/o all
4096->4096), 100-adapter catalog (20 per rank in {8,16,32,64,128}), one decode batch of
256 tokens with adapters drawn by the reference's assign_adapter(default_rng(seed)).
A step = the device segment-table build (K4) + LoRA apply for all 32 layers x 4 projections
(q/k/v fused into one launch over their shared input, o separate), replayed as one CUDA graph.
Synthetic random-init adapters (pool pages filled with N(0, 0.02) bf16) and activations.

value    = tokens/s over all ranks, inputs resident in HBM (max over ranks of the CUDA-event time)
e2e      = tokens/s through LoraStepExecutor with host buffers: every step's pinned H2D of the
           request table + hidden state, the step's graph, D2H of the last projection's output;
           wall clock over all steps, PCIe transfers overlapped with neighbouring steps
roofline = algorithmic bytes of the apply launches / their measured duration vs
           MEASURED_PEAKS.json hbm_gbs
cpu_baseline = the numpy oracle (oracle/lora_ref.py) on the host cores, bounded sample
--impl reference = that CPU path alone, on the same config/metric (the reference has no CPU
           LoRA implementation of its own — it only models the cost, engine.py:67-77).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "LoRA-apply tokens/sec and adapter-read HBM GB/s (% of peak), mixed ranks, 1/2/4/8 GPU"
H = 4096
N_LAYERS = 32
N_PROJ = 4
T_DECODE = 256
NUM_ADAPTERS = 100


WORKLOAD_C2 = ("C2: Llama-2-7B q/k/v/o LoRA (h=4096, 32 layers), 100 adapters ranks 8-128, "
               "decode batch 256 tokens per GPU (assign_adapter seed = rank)")
WORKLOAD_C3 = ("C3: Llama-2-7B q/k/v/o LoRA (h=4096, 32 layers) prefill, 64 segments x 64 tokens over "
               "64 adapters with power-law ranks (prefill_batch seed = rank), tcgen05 path")


L2_NOTE = ("inputs larger than L2: each step streams every distinct adapter's pages for all 128 "
           "(layer, proj) blocks (8 GB at C2) through the 126 MB L2")


def c2_config(world: int, mode: str) -> dict:
    """The C2 `config` object, printed identically by both arms (the driver's same_config)."""
    return {"workload": WORKLOAD_C2, "global_batch": T_DECODE * world, "seq_len": 1,
            "parallelism": f"replicas x{world}", "launch_mode": mode, "l2": L2_NOTE}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1681.7)), "measured"
    return 6650.0, 1590.0, "fallback"


def step_bytes(seg_off, seg_slot, seg_rank, n_tokens, h, es, n_layers, groups):
    """Algorithmic bytes of one step, counting x ONCE per launch group: every
    distinct adapter's A and B once per (layer, proj), y read + written once per (layer, proj),
    and x read once per (layer, projection group) — a fused q/k/v launch stages the shared
    input once for its three projections.  Returns (total, adapter part)."""
    a_lp, _ = algorithmic_bytes(seg_off, seg_slot, seg_rank, n_tokens, h, h, es)
    n_proj = sum(len(g) for g in groups)
    adapter = a_lp * n_proj * n_layers
    act = n_layers * (len(groups) * n_tokens * h * es + n_proj * 2 * n_tokens * h * es)
    return adapter + act, adapter


def algorithmic_bytes(seg_off, seg_slot, seg_rank, n_tokens, h_in, h_out, es):
    """SURVEY §8(d) per (layer, proj): every distinct adapter once (A and B) plus
    T * (h_in reads of x + h_out reads and writes of y)."""
    distinct = {}
    for i in range(len(seg_slot)):
        if seg_slot[i] >= 0 and seg_off[i + 1] > seg_off[i]:
            distinct[int(seg_slot[i])] = int(seg_rank[i])
    adapter = sum(r * (h_in + h_out) * es for r in distinct.values())
    act = n_tokens * (h_in + 2 * h_out) * es
    return adapter, act


def traffic_per_launch(config: str):
    """DRAM bytes per apply launch from the committed ncu --set full summary (scripts/ncu_summary.py),
    or None when no capture of this config is committed."""
    p = ROOT / "profiles" / f"traffic_{config}.json"
    if not p.exists():
        return None
    return float(json.loads(p.read_text())["traffic_per_launch"])


# --------------------------------------------------------------------------- clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._proc = None

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS"):  # fault-hunt experiments only
            return self
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except Exception:
                self._proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# --------------------------------------------------------------------------- CPU path
def cpu_oracle_sample(batch_ids, seconds: float = 12.0, ntok=None):
    """numpy fp32 restatement (oracle/lora_ref.py) of one (layer, proj) apply of the batch,
    repeated for ~`seconds`; returns (seconds per layer-proj, cores, sample description)."""
    from oracle.lora_ref import lora_apply_ref
    from oracle.segments_ref import build_segments_ref
    from paper_2411_17741_b200.workload import rank_of_id

    rng = np.random.default_rng(0)
    uniq = sorted(set(batch_ids))
    slot = {a: i for i, a in enumerate(uniq)}
    adapters = {}
    for a in uniq:
        r = rank_of_id(a)
        adapters[slot[a]] = ((rng.standard_normal((H, r)) * 0.02).astype(np.float32),
                             (rng.standard_normal((r, H)) * 0.02).astype(np.float32))
    ranks = [rank_of_id(a) for a in batch_ids]
    slots = [slot[a] for a in batch_ids]
    ntok = [1] * len(batch_ids) if ntok is None else [int(t) for t in ntok]
    perm, off, sl, rk = build_segments_ref(slots, ranks, ntok)
    x = rng.standard_normal((sum(ntok), H)).astype(np.float32)
    y = rng.standard_normal((sum(ntok), H)).astype(np.float32)
    n = 0
    t0 = time.perf_counter()
    while True:
        lora_apply_ref(x, y, perm, off, sl, rk, adapters, acc=np.float32)
        n += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = (time.perf_counter() - t0) / n
    cores = len(os.sched_getaffinity(0))
    return dt, cores, (f"{n} x one (layer,proj) apply of the batch ({sum(ntok)} tok, {len(uniq)} adapters), "
                       "numpy fp32")


def cpu_full_step(batch_ids, n_steps: int, n_warm: int = 1, weight_sets: int = 4):
    """The numpy fp32 restatement (oracle/lora_ref.py) of FULL steps: every (layer, proj) of the
    32 x 4 applies of the batch, each over its own adapter weights drawn from `weight_sets`
    rotating sets (4 x ~120 MB of distinct fp32 A/B, far beyond the host caches).  Returns
    (per-step seconds list, cores, sample description)."""
    from oracle.lora_ref import lora_apply_ref
    from oracle.segments_ref import build_segments_ref
    from paper_2411_17741_b200.workload import rank_of_id

    rng = np.random.default_rng(0)
    uniq = sorted(set(batch_ids))
    slot = {a: i for i, a in enumerate(uniq)}
    sets = []
    for _ in range(weight_sets):
        ad = {}
        for a in uniq:
            r = rank_of_id(a)
            ad[slot[a]] = ((rng.standard_normal((H, r)) * 0.02).astype(np.float32),
                           (rng.standard_normal((r, H)) * 0.02).astype(np.float32))
        sets.append(ad)
    ranks = [rank_of_id(a) for a in batch_ids]
    slots = [slot[a] for a in batch_ids]
    perm, off, sl, rk = build_segments_ref(slots, ranks, [1] * len(batch_ids))
    x = rng.standard_normal((len(batch_ids), H)).astype(np.float32)
    y = rng.standard_normal((len(batch_ids), H)).astype(np.float32)
    times = []
    for i in range(n_warm + n_steps):
        t0 = time.perf_counter()
        for lp in range(N_LAYERS * N_PROJ):
            lora_apply_ref(x, y, perm, off, sl, rk, sets[lp % weight_sets], acc=np.float32)
        if i >= n_warm:
            times.append(time.perf_counter() - t0)
    cores = len(os.sched_getaffinity(0))
    return times, cores, (f"full steps: 128 (layer,proj) applies of the batch ({len(batch_ids)} tok, {len(uniq)} "
                          f"adapters) over {weight_sets} rotating distinct weight sets, numpy fp32 (BLAS threads = "
                          f"{cores} cores)")


def decision_path_record():
    try:
        from bench_decisions import decision_path

        return decision_path()
    except Exception as e:  # the GPU line must not die on the CPU side-measurement
        return {"unavailable": f"{type(e).__name__}: {e}"}


def run_reference(args, rank: int, world: int):
    """The reference arm: the reference has no LoRA implementation of its own (it models the
    cost, engine.py:67-77), so its CPU path is the oracle port, timed over full C2 steps on all
    host cores; the reference's own decision path (baseline/_ref) is timed beside it."""
    if rank != 0:
        return
    from bench_decisions import cpu_model
    from paper_2411_17741_b200.workload import decode_batch

    batch = decode_batch(0, T_DECODE, NUM_ADAPTERS)
    n = max(1, min(args.steps, args.cpu_max_steps))
    times, cores, sample = cpu_full_step(batch, n, n_warm=1 if args.warmup > 0 else 0)
    step_s = statistics.median(times)
    value = T_DECODE / step_s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": n, "warmup": 1 if args.warmup > 0 else 0, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": c2_config(world, args.mode),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": sample + f"; median of {n} timed full steps (--steps {args.steps} capped at "
                                            f"--cpu-max-steps {args.cpu_max_steps})"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "decision_path": decision_path_record(),
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU path
def measure(config: str, args, rank: int, world: int, e2e: bool = True) -> dict:
    """Build the config's pool, batch and step graph on this rank's GPU and time it: K step
    replays (CUDA events, max over ranks), the apply-only graph (roofline), and optionally the
    host-buffer e2e loop.  Returns the raw measurements for the JSON line."""
    import torch
    import torch.distributed as dist

    from paper_2411_17741_b200.executor import LoraStepExecutor
    from paper_2411_17741_b200.model import build_catalog
    from paper_2411_17741_b200.pool import AdapterPool, pages_for_rank
    from paper_2411_17741_b200.workload import decode_batch, prefill_batch, rank_of_id

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    if config == "c3":
        # C3: 64 prefill segments x 64 tokens, one distinct adapter each (prefill_batch(seed=rank))
        pids, pntok = prefill_batch(rank)
        ids = list(dict.fromkeys(pids))
        rank_of = {a: rank_of_id(a) for a in ids}
        batch, ntok_list = pids, pntok
    else:
        catalog = build_catalog(NUM_ADAPTERS)
        ids = list(catalog)
        rank_of = {a: catalog[a].rank for a in ids}
        batch = decode_batch(rank, T_DECODE, NUM_ADAPTERS)
        ntok_list = [1] * len(batch)
    slot_of = {a: i for i, a in enumerate(ids)}
    n_pages = sum(pages_for_rank(rank_of[a]) for a in ids)
    pool = AdapterPool(n_pages, N_LAYERS, [H] * N_PROJ, [H] * N_PROJ, dtype=torch.bfloat16,
                       n_slots=len(ids), max_tokens=4096, device=dev)
    # synthetic random-init adapters: every page of every adapter gets N(0, 0.02) bf16 values
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    page = 0
    for a in ids:
        r = rank_of[a]
        npg = pages_for_rank(r)
        pool.set_slot(slot_of[a], r, list(range(page, page + npg)))
        buf = (torch.randn(npg * pool.page_bytes // 2, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
        pool.fill_from_device(slot_of[a], buf.view(torch.uint8))
        page += npg
        del buf
    torch.cuda.synchronize(dev)

    req_slot = np.array([slot_of[a] for a in batch], dtype=np.int32)
    req_rank = np.array([rank_of[a] for a in batch], dtype=np.int32)
    req_ntok = np.array(ntok_list, dtype=np.int32)

    groups = [[0, 1, 2], [3]] if args.mode == "qkv" else [[0], [1], [2], [3]]
    ex = LoraStepExecutor(pool, max_requests=1024, max_tokens=4096, proj_groups=groups)
    T = int(req_ntok.sum())
    xs = [[torch.randn(T, H, device=dev).to(torch.bfloat16) for _ in groups] for _ in range(N_LAYERS)]
    ys = [[torch.randn(T, H, device=dev).to(torch.bfloat16) for _ in range(N_PROJ)] for _ in range(N_LAYERS)]
    ex.upload(req_slot, req_rank, req_ntok)
    torch.cuda.synchronize(dev)

    s = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s):
        ex.run(xs, ys)  # eager warm-up (sets kernel attributes before capture)
    torch.cuda.synchronize(dev)
    g_step = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_step, stream=s):
        ex.run(xs, ys)
    g_apply = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_apply, stream=s):
        for layer in range(N_LAYERS):
            ex.apply_layer(layer, xs[layer], ys[layer])
    torch.cuda.synchronize(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- timed region: K step replays, inputs resident in HBM
    with torch.cuda.stream(s):
        for _ in range(args.warmup):
            g_step.replay()
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # clocks are sampled (every 20 ms) over the whole GPU measurement: the timed steps, the
    # apply-only replays and the e2e loop
    clk = ClockSampler(dev.index).__enter__()
    with torch.cuda.stream(s):
        ev0.record(s)
        for _ in range(args.steps):
            g_step.replay()
        ev1.record(s)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    step_ms = ev0.elapsed_time(ev1) / args.steps
    # apply-only graph for the roofline (the apply kernels launch alone), at least ~200 ms of
    # replays so the clock sampler sees the load
    reps = max(args.steps, int(200.0 / max(step_ms, 1e-3)) + 1)
    with torch.cuda.stream(s):
        ev0.record(s)
        for _ in range(reps):
            g_apply.replay()
        ev1.record(s)
    torch.cuda.synchronize(dev)
    apply_ms = ev0.elapsed_time(ev1) / reps
    step_ms = max_over_ranks(step_ms)
    apply_ms = max_over_ranks(apply_ms)

    # ---- e2e: through the executor with host buffers (pinned H2D request table + hidden
    #      state, step graph, D2H of the last projection's output), wall clock over the steps
    #      Pipelined like a serving loop: the host enqueues step i+1 while step i runs, and the
    #      PCIe transfers run on a copy stream: step i+1's input H2D and step i-1's output D2H
    #      overlap step i's kernels (double-buffered device staging, event-ordered reuse).
    x_host = torch.randn(T, H).to(torch.bfloat16).pin_memory()
    y_host = [torch.empty(T, H, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    h2d = 3 * len(batch) * 4 + x_host.numel() * 2
    d2h = y_host[0].numel() * 2
    cs = torch.cuda.Stream(device=dev)
    x_stage = [torch.empty(T, H, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    y_stage = [torch.empty(T, H, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    ev_x, ev_xfree, ev_y, ev_yfree = [None, None], [None, None], [None, None], [None, None]
    ev_up = None

    def record(stream):
        e = torch.cuda.Event()
        e.record(stream)
        return e

    def stage_input(b):  # this step's hidden state: pinned host -> device staging, copy stream
        with torch.cuda.stream(cs):
            if ev_xfree[b] is not None:
                cs.wait_event(ev_xfree[b])
            x_stage[b].copy_(x_host, non_blocking=True)
            ev_x[b] = record(cs)

    n_total = args.warmup + args.steps if e2e and not os.environ.get("BENCH_NO_E2E") else 0
    e2e_s = None
    if n_total:
        stage_input(0)
        t0 = time.perf_counter()
        for i in range(n_total):
            if i == args.warmup:
                s.synchronize()
                cs.synchronize()
                barrier()
                t0 = time.perf_counter()
                stage_input(i & 1)  # this step's input transfer belongs to the timed region
            b = i & 1
            if i + 1 < n_total:
                stage_input(b ^ 1)  # the next step's input streams in while this step computes
            if ev_up is not None:
                ev_up.synchronize()  # the pinned request staging was consumed by the previous upload
            with torch.cuda.stream(s):
                s.wait_event(ev_x[b])
                xs[0][0].copy_(x_stage[b])
                ev_xfree[b] = record(s)
                ex.upload(req_slot, req_rank, req_ntok, stream=s)
                ev_up = record(s)
                if ev_yfree[b] is not None:
                    s.wait_event(ev_yfree[b])
                g_step.replay()
                y_stage[b].copy_(ys[N_LAYERS - 1][N_PROJ - 1])
                ev_y[b] = record(s)
            with torch.cuda.stream(cs):
                cs.wait_event(ev_y[b])
                y_host[b].copy_(y_stage[b], non_blocking=True)  # the step's result to the host
                ev_yfree[b] = record(cs)
        s.synchronize()
        cs.synchronize()
        e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
    clk.__exit__()
    err = pool.device_error(clear=True, stream=s)  # 0: no kernel met a device-side limit

    # ---- algorithmic bytes / flops from the rank's segment table
    perm, off, sl, rk = ex.table.to_host()
    lp = N_LAYERS * N_PROJ
    bytes_step, adapter_bytes_step = step_bytes(off, sl, rk, T, H, 2, N_LAYERS, groups)
    flops_step = int(2 * sum(int(rk[i]) * int(off[i + 1] - off[i]) for i in range(len(sl))) * (H + H) * lp)
    out = {"T": T, "batch": batch, "req_ntok": req_ntok, "groups": groups, "step_ms": step_ms,
           "apply_ms": apply_ms, "e2e_s": e2e_s, "h2d": h2d, "d2h": d2h, "bytes_step": int(bytes_step),
           "adapter_bytes_step": int(adapter_bytes_step), "flops_step": flops_step,
           "launches_per_step": ex.launches_per_step(), "apply_launches": N_LAYERS * len(groups),
           "clocks": clk.summary(), "device_error": err}
    pool.close()
    del xs, ys, ex, g_step, g_apply
    torch.cuda.empty_cache()
    return out


def sub_record(config: str, args, rank: int, world: int) -> dict:
    """C4 (cache with misses) / C5 (70B dims, TP = world) measured in the same driver run as the
    C2 line, with short step counts; a failure is recorded, never fatal to the headline line."""
    import copy

    import torch

    a = copy.copy(args)
    a.steps, a.warmup = (20, 3) if config == "c4" else (10, 3)
    try:
        line = (run_c4 if config == "c4" else run_c5)(a, rank, world, emit=False)
    except Exception as e:  # pragma: no cover - reported in the line
        torch.cuda.synchronize()
        return {"error": f"{type(e).__name__}: {e}"[:300]}
    finally:
        torch.cuda.empty_cache()
    keep = ("value", "unit", "ms_per_step", "steps", "warmup", "config", "roofline", "cache", "decisions",
            "adapter_read_gbs_per_rank", "gpu_launches", "clocks", "device_error")
    return {k: line[k] for k in keep if k in line}


def roofline_record(m: dict, config: str) -> dict:
    hbm_peak, bf16_peak, peak_kind = peaks()
    achieved = m["bytes_step"] / (m["apply_ms"] * 1e-3) / 1e9
    if config == "c3":
        kernel = ("prefill::fused_kernel (tcgen05, TMEM accumulators; shrink -> per-tile V images -> expand, "
                  "PDL-chained) per apply")
    else:
        kernel = ("decode::lora_apply_kernel<bf16> (shrink and expand units from one queue, per-tile v-ready "
                  "counters, PDL-chained)")
    return {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved / hbm_peak, "peak_kind": peak_kind, "kernel": kernel,
            "bytes_per_step": m["bytes_step"],
            "bytes_formula": "SURVEY 8(d) per (layer, proj): distinct adapters' A+B once, y read+write; "
                             "x once per launch group (q/k/v share one staged input)",
            "launches_per_step": m["apply_launches"],
            "algorithmic_bytes_per_launch": m["bytes_step"] / m["apply_launches"],
            "avg_launch_us": m["apply_ms"] * 1e3 / m["apply_launches"],
            "traffic": traffic_per_launch(config),
            "traffic_source": "profiles/traffic_%s.json (ncu --set full, cold L2, DRAM read+write "
                              "bytes per launch, mean of one q/k/v and one o launch)" % config}


def run_ours(args, rank: int, world: int):
    m = measure(args.config, args, rank, world, e2e=True)
    c3 = None
    if args.config == "c2" and not args.no_c3:
        # the tcgen05 prefill path measured in the same driver run (C3 sub-record, no e2e loop)
        c3 = measure("c3", args, rank, world, e2e=False)
    if rank != 0:
        return
    hbm_peak, bf16_peak, _ = peaks()
    T = m["T"]
    tokens_total = T * world
    value = tokens_total / (m["step_ms"] * 1e-3)
    if args.config == "c3":
        config = {"workload": WORKLOAD_C3, "global_batch": tokens_total, "seq_len": int(m["req_ntok"].max()),
                  "parallelism": f"replicas x{world}", "launch_mode": args.mode,
                  "l2": "inputs larger than L2: each step streams 16.8 GB of activations and adapter pages"}
    else:
        config = c2_config(world, args.mode)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["step_ms"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": config,
        "adapter_read_gbs": m["adapter_bytes_step"] / (m["step_ms"] * 1e-3) / 1e9,
        "adapter_read_frac_of_peak": m["adapter_bytes_step"] / (m["step_ms"] * 1e-3) / 1e9 / hbm_peak,
        "roofline": roofline_record(m, args.config),
        "flops_per_step": m["flops_step"],
        "tensor_frac_of_peak": m["flops_step"] / (m["apply_ms"] * 1e-3) / 1e12 / bf16_peak,
        "e2e": {"value": tokens_total / m["e2e_s"], "unit": "tokens/s", "h2d_bytes_per_step": m["h2d"],
                "d2h_bytes_per_step": m["d2h"], "ms_per_step": m["e2e_s"] * 1e3,
                "mode": "every step: LoraStepExecutor.upload (pinned H2D of the request table), pinned H2D of "
                        "the hidden state and pinned D2H of the output on a copy stream overlapping the "
                        "neighbouring steps' kernels, step graph; wall clock over all steps"},
        "gpu_launches": args.steps * m["launches_per_step"],
        "clocks": m["clocks"],
        "device_error": m["device_error"],
    }
    if c3 is not None:
        line["c3"] = {
            "workload": WORKLOAD_C3, "tokens_s": c3["T"] * world / (c3["step_ms"] * 1e-3),
            "ms_per_step": c3["step_ms"], "steps": args.steps, "warmup": args.warmup,
            "roofline": roofline_record(c3, "c3"),
            "tensor_frac_of_peak": c3["flops_step"] / (c3["apply_ms"] * 1e-3) / 1e12 / bf16_peak,
            "clocks": c3["clocks"], "device_error": c3["device_error"],
            "gpu_launches": args.steps * c3["launches_per_step"]}
        line["gpu_launches"] += line["c3"]["gpu_launches"]
    if args.config == "c2" and world == 1 and not args.no_subrecords:
        line["c4"] = sub_record("c4", args, rank, world)
        line["c5"] = sub_record("c5", args, rank, world)
        for k in ("c4", "c5"):
            line["gpu_launches"] += line[k].get("gpu_launches", 0) if isinstance(line[k], dict) else 0
    if world == 1 and not args.no_cpu_baseline:
        from bench_decisions import cpu_model

        lp = N_LAYERS * N_PROJ
        t_lp, cores, sample = cpu_oracle_sample(m["batch"], seconds=args.cpu_seconds, ntok=list(m["req_ntok"]))
        line["cpu_baseline"] = {"value": T / (t_lp * lp), "unit": "tokens/s", "cores": cores, "kind": "port",
                                "cpu_model": cpu_model(),
                                "sample": sample + f"; tokens/s = {T} / (128 x that); the --impl reference "
                                                   "arm times full 128-apply steps"}
        line["decision_path"] = decision_path_record()
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- C4: cache with misses
def run_c4(args, rank: int, world: int, emit: bool = True):
    """C4 replica: 1000-adapter Zipf(0.7) catalog, PagedAdapterCache at 10% of idle HBM, a
    closed loop of 256 decode requests (each step's zipf draws, seeded by replica rank and
    step, replace the requests the previous step executed), admitted up to 256 per step.  A step is `serving.ReplicaLoop.step`: fill completions by
    poll_fills (engine.py:294-301), the reference's admission transaction with real pinned
    fills on the side stream for misses (engine.py:491-532), queue-driven prefetch of the
    queued requests' adapters (engine.py:457-470), then the step graph (K4 + plan + 64
    applies) over every ready request, ordered after its fills on the device.  Timed by wall
    clock around all steps (host decisions and PCIe fills included).  After the run the
    replica's recorded decision trace is replayed through a fresh AdapterCache (bit-exact
    with the reference's, tests/test_cache.py) and every decision must match."""
    import torch
    import torch.distributed as dist

    from paper_2411_17741_b200.adapter_cache import AdapterCache, PagedAdapterCache
    from paper_2411_17741_b200.executor import LoraStepExecutor
    from paper_2411_17741_b200.model import CacheConfig, PrefetchMode, make_adapter_spec, zipf_catalog
    from paper_2411_17741_b200.pool import AdapterPool, pages_for_rank
    from paper_2411_17741_b200.serving import ReplicaLoop, replay_ops

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    ids, probs = zipf_catalog(1000)
    catalog = {a: make_adapter_spec(a, int(a[1:].split("-")[0])) for a in ids}
    free_b, _ = torch.cuda.mem_get_info(dev)
    page_bytes = N_LAYERS * N_PROJ * 8 * (H + H) * 2
    n_pages = int(0.10 * free_b) // page_bytes
    pool = AdapterPool(n_pages, N_LAYERS, [H] * N_PROJ, [H] * N_PROJ, dtype=torch.bfloat16, n_slots=len(ids),
                       max_tokens=4096, device=dev)
    # host repository: one pinned synthetic packed adapter per rank class (the content of a
    # synthetic adapter does not change the bytes moved); N(0, 0.02) bf16
    by_rank = {}
    for r in sorted({c.rank for c in catalog.values()}):
        by_rank[r] = (torch.randn(pages_for_rank(r) * page_bytes // 2) * 0.02).to(torch.bfloat16).view(
            torch.uint8).pin_memory()
    store = {a: by_rank[catalog[a].rank] for a in ids}
    s = torch.cuda.Stream(device=dev)
    prefetch = PrefetchMode.OFF if args.no_prefetch else PrefetchMode.QUEUE_DRIVEN
    cfg = CacheConfig(prefetch=prefetch)
    cache = PagedAdapterCache(cfg, catalog, pool, host_store=store, compute_stream=s)
    groups = [[0, 1, 2], [3]]
    max_req = 1024
    ex = LoraStepExecutor(pool, max_requests=max_req, max_tokens=max_req, proj_groups=groups,
                          graph_requests=max_req)
    xs = [[torch.randn(max_req, H, device=dev).to(torch.bfloat16) for _ in groups] for _ in range(N_LAYERS)]
    ys = [[torch.randn(max_req, H, device=dev).to(torch.bfloat16) for _ in range(N_PROJ)] for _ in range(N_LAYERS)]
    state = {"graph": False, "batches": 0, "tokens": 0}

    def run_batch(slots, ranks, ntok):
        for lo in range(0, len(slots), max_req):
            sl, rk, nt = slots[lo:lo + max_req], ranks[lo:lo + max_req], ntok[lo:lo + max_req]
            ex.upload(sl, rk, nt, stream=s)
            if not state["graph"]:
                ex.capture(xs, ys, s)
                state["graph"] = True
            ex.replay()
            state["batches"] += 1
            state["tokens"] += int(nt.sum())

    loop = ReplicaLoop(cache, catalog, run_batch, capacity_tokens=n_pages * PagedAdapterCache.TOKENS_PER_PAGE,
                       max_admit=T_DECODE)
    p = np.asarray(probs)

    def arrivals(i):
        # closed loop at 256 requests in the replica: new arrivals replace the requests the
        # previous step executed (queued and fill-waiting requests stay in the system)
        n = T_DECODE - len(loop.deferred) - sum(loop.waiters.values())
        rng = np.random.default_rng(rank * 1_000_003 + i)
        return [ids[int(k)] for k in rng.choice(len(ids), max(0, n), p=p)]

    n_warm = args.warmup * 4
    for i in range(n_warm):  # warm the cache towards its steady state
        loop.step(arrivals(i))
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    st0 = dict(loop.stats)
    h0, m0, l0, ev0, fb0, tok0 = cache.hits, cache.misses, cache.loads, cache.evictions, cache.fill_bytes, \
        state["tokens"]
    t0 = time.perf_counter()
    with ClockSampler(dev.index) as clk:
        for i in range(args.steps):
            loop.step(arrivals(n_warm + i))
        torch.cuda.synchronize(dev)
    el = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([el], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    hits, misses = cache.hits - h0, cache.misses - m0
    fill_b = cache.fill_bytes - fb0
    tokens_rank = state["tokens"] - tok0
    err = pool.device_error(clear=True, stream=s)
    # decision parity: the replica's whole trace (warm-up included) through a fresh cache
    t_rep = time.perf_counter()
    mism = replay_ops(AdapterCache(cfg, catalog), cache.op_log)
    t_rep = time.perf_counter() - t_rep
    # PCIe fill bandwidth alone: the largest adapter copied 5 times on the side stream
    big = by_rank[max(by_rank)]
    scratch = torch.empty(big.numel(), dtype=torch.uint8, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cache.fill_stream):
        e0.record()
        for _ in range(5):
            scratch.copy_(big, non_blocking=True)
        e1.record()
    torch.cuda.synchronize(dev)
    fill_gbs = 5 * big.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9
    tok = torch.tensor([tokens_rank], dtype=torch.float64, device=dev if world > 1 and dist.get_backend() == "nccl"
                       else "cpu")
    if world > 1:
        dist.all_reduce(tok, op=dist.ReduceOp.SUM)
    tokens = float(tok.item())
    if rank == 0:
        d = {k: loop.stats[k] - st0[k] for k in loop.stats}
        line = {
            "metric": METRIC, "value": tokens / el, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": n_warm, "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (one pinned random adapter image per rank class)",
            "config": {"workload": "C4: 1000 adapters Zipf(0.7), PagedAdapterCache at 10% of idle HBM "
                                   f"({n_pages} pages = {n_pages * page_bytes / 1e9:.1f} GB), closed loop of 256 decode "
                                   "requests (Zipf draws replace the executed ones every step), misses filled over "
                                   f"PCIe on a side stream, prefetch {enum_name(prefetch)}",
                       "global_batch": T_DECODE * world, "seq_len": 1, "parallelism": f"replicas x{world}",
                       "timing": "wall clock incl. host cache decisions, fills and the step graphs"},
            "cache": {"hit_rate": hits / max(1, hits + misses), "hits": hits, "misses": misses,
                      "loads": cache.loads - l0, "evictions": cache.evictions - ev0,
                      "prefetches": d["prefetches"], "prefetch_hits": d["prefetch_hits"],
                      "joined_inflight": d["joined"], "queued_request_steps": d["deferred"],
                      "executed_requests": d["executed"],
                      "fill_bytes_per_step": fill_b / args.steps, "fill_gbs_during_run": fill_b / el / 1e9,
                      "pcie_fill_gbs_alone": fill_gbs, "host_blocked_on_fills_s": 0.0},
            "decisions": {"ops": len(cache.op_log), "mismatches": len(mism), "replay_s": t_rep,
                          "checked_against": "fresh AdapterCache (bit-exact with the reference's, "
                                             "tests/test_cache.py + tests/test_replica.py)"},
            "device_error": err,
            "gpu_launches": state["batches"] * ex.launches_per_step(),
            "clocks": clk.summary(),
        }
        if emit:
            print(json.dumps(line), flush=True)
        pool.close()
        return line
    pool.close()
    return None


def enum_name(v):
    return getattr(v, "value", v)



# --------------------------------------------------------------------------- C5: tensor parallel
H70, L70 = 8192, 80
H70_IN = [8192, 8192, 8192, 8192]   # q, k, v, o
H70_OUT = [8192, 1024, 1024, 8192]  # GQA: 8 KV heads
C5_ADAPTERS, C5_RANK = 100, 64


def run_c5(args, rank: int, world: int, emit: bool = True):
    """C5: Llama-2-70B dims (80 layers; q/o 8192->8192, k/v 8192->1024), 100 adapters of rank 64,
    decode batch of 256 tokens, tensor parallel over the N ranks (TP = N; every rank sees the
    same tokens).  A step = per layer: shrink of the rank's x shard for q/k/v into one fused
    [T, 3 x 64] fp32 v, ONE all-reduce of it, expand into the rank's y shards; then the same for
    o (its own all-reduce): 160 all-reduces per step at N > 1 (tp.py).  At TP
    degree 1 there is no exchange step and TensorParallelLora runs the fused apply instead (q,
    k+v, o: 3 launches per layer).  The step is one CUDA graph (NCCL all-reduces captured);
    value = tokens/s of the TP group."""
    import torch
    import torch.distributed as dist

    from paper_2411_17741_b200.executor import segment_token_bounds
    from paper_2411_17741_b200.ops import build_plan, build_segments
    from paper_2411_17741_b200.pool import AdapterPool, pages_for_rank
    from paper_2411_17741_b200.tp import TensorParallelLora, shard_dims

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    hin_l, hout_l = shard_dims(H70_IN, H70_OUT, world)
    npg = pages_for_rank(C5_RANK)
    pool = AdapterPool(C5_ADAPTERS * npg, L70, hin_l, hout_l, dtype=torch.bfloat16, n_slots=C5_ADAPTERS,
                       max_tokens=T_DECODE, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321 + rank)
    for a in range(C5_ADAPTERS):
        pool.set_slot(a, C5_RANK, list(range(a * npg, (a + 1) * npg)))
        buf = (torch.randn(npg * pool.page_bytes // 2, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
        pool.fill_from_device(a, buf.view(torch.uint8))
        del buf
    torch.cuda.synchronize(dev)
    # the same decode batch on every TP rank: 256 requests, adapters uniform over the catalog
    req_slot = np.random.default_rng(0).integers(0, C5_ADAPTERS, T_DECODE).astype(np.int32)
    req_rank = np.full(T_DECODE, C5_RANK, dtype=np.int32)
    # host routing hints (as LoraStepExecutor.upload passes them): every segment is decode-sized,
    # so no launch of the step needs the prefill kernel family
    lo, hi = segment_token_bounds(req_slot, req_rank, np.ones(T_DECODE, dtype=np.int32))
    pool.set_prefill_route(64, lo, hi)
    table = build_segments(req_slot, req_rank, np.ones(T_DECODE, dtype=np.int32), device=dev)
    n_seg = int(table.n_seg.item())
    table.n_seg_host = n_seg
    build_plan(table, pool=pool)
    groups = [[0, 1, 2], [3]]
    group = dist.group.WORLD if world > 1 else False
    tp = TensorParallelLora(pool, max_tokens=T_DECODE, r_stride=C5_RANK, proj_groups=groups, group=group, device=dev)
    xs = [[torch.randn(T_DECODE, hin_l[g[0]], device=dev).to(torch.bfloat16) for g in groups] for _ in range(L70)]
    ys = [[torch.randn(T_DECODE, hout_l[p], device=dev).to(torch.bfloat16) for p in range(4)] for _ in range(L70)]
    kw = dict(perm=table.perm[:T_DECODE], n_positions=T_DECODE, plan=table.plan)

    def step(stream):
        for layer in range(L70):
            for gi, projs in enumerate(groups):
                tp.apply_group(layer, projs, xs[layer][gi], [ys[layer][p] for p in projs],
                               table.seg_slot[:n_seg], table.seg_off[:n_seg + 1], table.seg_rank[:n_seg],
                               stream=stream, **kw)

    s = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s):
        step(s)  # eager warm-up (kernel attributes, NCCL communicator)
    torch.cuda.synchronize(dev)
    graph = None
    if world == 1 or dist.get_backend() == "nccl":
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            step(s)
        torch.cuda.synchronize(dev)

    def run_steps(n):
        with torch.cuda.stream(s):
            for _ in range(n):
                if graph is not None:
                    graph.replay()
                else:
                    step(s)

    run_steps(args.warmup)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        ev0.record(s)
        run_steps(args.steps)
        ev1.record(s)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
    step_ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([step_ms], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms = float(t.item())
    # algorithmic bytes of this rank's shard (SURVEY §8d per (layer, proj), local dims)
    perm, off, sl, rk = table.to_host()
    bytes_rank = 0
    adapter_rank = 0
    for p in range(4):
        a_b, act_b = algorithmic_bytes(off, sl, rk, T_DECODE, hin_l[p], hout_l[p], 2)
        bytes_rank += (int(a_b) + int(act_b)) * L70
        adapter_rank += int(a_b) * L70
    hbm_peak, _, peak_kind = peaks()
    achieved = bytes_rank / (step_ms * 1e-3) / 1e9
    if rank == 0:
        distinct = len(set(req_slot.tolist()))
        line = {
            "metric": METRIC, "value": T_DECODE / (step_ms * 1e-3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"C5: Llama-2-70B dims LoRA (80 layers, q/o 8192->8192, k/v 8192->1024), "
                                   f"{C5_ADAPTERS} adapters of rank {C5_RANK} ({distinct} distinct in the batch), "
                                   f"decode batch {T_DECODE} tokens, TP={world}",
                       "global_batch": T_DECODE, "seq_len": 1, "parallelism": f"tp{world}",
                       "collectives_per_step": 2 * L70 if world > 1 else 0,
                       "l2": "inputs larger than L2: each step streams the shards of every distinct adapter"},
            "adapter_read_gbs_per_rank": adapter_rank / (step_ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                         "kernel": ("decode::lora_apply_kernel<bf16> MODE_SHRINK / MODE_EXPAND around the all-reduce "
                                    "(rank 0's step incl. collectives)") if world > 1 else
                                   "decode::lora_apply_kernel<bf16> fused (TP degree 1: no exchange, q and k+v and o "
                                   "launches)",
                         "bytes_per_step_per_rank": bytes_rank, "launches_per_step": L70 * (5 if world > 1 else 3)},
            "gpu_launches": args.steps * L70 * (5 if world > 1 else 3),
            "clocks": clk.summary(),
        }
        if emit:
            print(json.dumps(line), flush=True)
        pool.close()
        return line
    pool.close()
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["qkv", "per-proj"], default="qkv")
    ap.add_argument("--config", choices=["c2", "c3", "c4", "c5"], default="c2",
                    help="c2 (default, the BASELINE metric's decode config) or c3 (prefill, tcgen05 path)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--cpu-max-steps", type=int, default=8,
                    help="reference arm: full CPU steps timed (each ~2 s on 16 cores)")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 (tcgen05 prefill) sub-record")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prefetch", action="store_true", help="C4: prefetch off (the reference's default)")
    ap.add_argument("--no-subrecords", action="store_true", help="C2 line without the C4/C5 sub-records")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count()))
        # NCCL for the timing plumbing (the data path has no collective: replicas); gloo for the
        # CPU reference arm, or by BENCH_DIST_BACKEND (e.g. several ranks sharing one GPU in a test)
        backend = os.environ.get("BENCH_DIST_BACKEND") or ("gloo" if args.impl == "reference" else "nccl")
        dist.init_process_group(backend=backend)
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        elif args.config == "c4":
            run_c4(args, rank, world)
        elif args.config == "c5":
            run_c5(args, rank, world)
        else:
            run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
