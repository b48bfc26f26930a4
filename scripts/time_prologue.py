"""Times the step prologue kernels on the C2 batch: K4 (segment table) and the launch plan,
each alone and together, as CUDA graphs of 200 back-to-back launches (per-launch us)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_17741_b200.executor import LoraStepExecutor  # noqa: E402
from paper_2411_17741_b200.model import build_catalog  # noqa: E402
from paper_2411_17741_b200.ops import build_plan, build_segments  # noqa: E402
from paper_2411_17741_b200.pool import AdapterPool, pages_for_rank  # noqa: E402
from paper_2411_17741_b200.workload import decode_batch  # noqa: E402

cat = build_catalog(100)
ids = list(cat)
slot_of = {a: i for i, a in enumerate(ids)}
n_pages = sum(pages_for_rank(cat[a].rank) for a in ids)
pool = AdapterPool(n_pages, 1, [4096] * 4, [4096] * 4, dtype=torch.bfloat16, n_slots=len(ids), max_tokens=4096)
page = 0
for a in ids:
    npg = pages_for_rank(cat[a].rank)
    pool.set_slot(slot_of[a], cat[a].rank, list(range(page, page + npg)))
    page += npg
batch = decode_batch(0, 256, 100)
ex = LoraStepExecutor(pool, max_requests=1024, max_tokens=4096, proj_groups=[[0, 1, 2], [3]])
ex.upload(np.array([slot_of[a] for a in batch], np.int32), np.array([cat[a].rank for a in batch], np.int32),
          np.ones(256, np.int32))
torch.cuda.synchronize()
s = torch.cuda.Stream()
n = ex.n_req


def k4():
    build_segments(ex.req_dev[0, :n], ex.req_dev[1, :n], ex.req_dev[2, :n], device=pool.device, out=ex.table)


def plan():
    build_plan(ex.table, pool=pool)


for name, fn in [("k4", k4), ("plan", plan), ("k4+plan", lambda: (k4(), plan()))]:
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(200):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(5):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) * 1e3 / 1000:.2f} us per launch (group)")
