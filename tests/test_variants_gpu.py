"""The prefill kernel's experiment switches that are off by default stay correct.

`CHAM_PF_LD2=1` (two loader warps in the expand phase) and `CHAM_PF_SPLITX=1` (shrink-only
fused kernel + standalone expand kernel) lost their A/B on C3 (DESIGN.md §6 item 3) but are
kept as switches; this builds each variant library into build/variants/ and runs the small
decode + prefill parity check (scripts/sanitize_small.py, checked against the oracle) on it,
plus the chained two-layer executor check on the two-loader build.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

VARIANTS = {
    "t_ld2": ("CHAM_PF_LD2=1",),
    "t_splitx": ("CHAM_PF_SPLITX=1",),
}


def _variant(name):
    from paper_2411_17741_b200.csrc.build import build

    out = ROOT / "build" / "variants" / f"{name}.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    return build(force=True, out=out, defines=VARIANTS[name])


def _run(lib, args, timeout=600):
    env = dict(os.environ, CHAM_LIB=str(lib))
    r = subprocess.run([sys.executable, *args], cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, f"{args} on {lib.name}:\n{r.stdout[-2000:]}\n{r.stderr[-2000:]}"
    return r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_prefill_variant_matches_oracle(name):
    lib = _variant(name)
    out = _run(lib, ["scripts/sanitize_small.py"])
    assert "match the oracle" in out


@pytest.mark.gpu
def test_two_loader_variant_executor_chain():
    lib = _variant("t_ld2")
    _run(lib, ["-m", "pytest", "-q", "-m", "gpu", "-x", "tests/test_executor_gpu.py::test_c3_full_4096_tokens_two_layers",
               "tests/test_executor_gpu.py::test_executor_multilayer_qkv_o_decode_and_mixed"], timeout=900)
