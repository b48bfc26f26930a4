"""bench.py's multi-process path on one GPU (the driver runs it on N GPUs under torchrun): two
ranks sharing cuda:0 over gloo must print exactly ONE contract line from rank 0 with
n_gpus = 2 — C2 and C4 as independent replicas (no data-path collective), C5 as
TP=2 with the all-reduce of the shrink output."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config", ["c2", "c4", "c5"])
def test_two_rank_bench_prints_one_line(config):
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", BENCH_NO_CLOCKS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + ["c2", "c4", "c5"].index(config)),
           str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", config,
           "--no-c3", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["unit"] == "tokens/s"
    assert d.get("device_error", 0) == 0
    if config == "c4":
        assert d["decisions"]["mismatches"] == 0 and d["decisions"]["ops"] > 0
    if config == "c5":
        assert d["config"]["parallelism"] == "tp2" and d["config"]["collectives_per_step"] == 160
    else:
        assert d["scaling"] == "weak" and d["config"]["parallelism"] == "replicas x2"
