"""GPU box: run the random mixed-batch parity check (tests/test_prefill_gpu.py::_fuzz) over many
seeds; prints failures.  usage: python scripts/fuzz_sweep.py [n_seeds]"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import test_prefill_gpu as t  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
bad = 0
for seed in range(1000, 1000 + n):
    for dtype in (torch.bfloat16, torch.float32):
        try:
            t._fuzz(seed, dtype)
        except AssertionError as e:
            bad += 1
            print("MISMATCH seed", seed, dtype, str(e).splitlines()[:6], flush=True)
print(f"fuzz sweep: {2 * n} cases, {bad} mismatches")
