"""The C-ABI boundary without a GPU: the in-tree .so loads, exports exactly what
include/chameleon_lora.h declares (and _lib binds), reports its limits, fails with a status
code (no crash) when no device is present, and packs adapters bit-exactly in the page
layout the numpy oracle restates (oracle/pool_ref.py)."""
import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle.lora_ref import bf16_bits, bf16_round
from oracle.pool_ref import geometry, pack_adapter, unpack_block
from paper_2411_17741_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "chameleon_lora.h"


@pytest.fixture(scope="module")
def lib():
    if not _lib.LIB_PATH.exists():
        from paper_2411_17741_b200.csrc.build import build

        build()
    return _lib.lib()


def header_symbols():
    return sorted(set(re.findall(r"CHAM_API\s+[\w\s\*]+?\b(cham_\w+)\s*\(", HEADER.read_text())))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for s in ("cham_pool_create", "cham_pool_fill_async", "cham_build_segments", "cham_lora_apply",
              "cham_lora_shrink", "cham_lora_expand"):
        assert s in syms
    assert sorted(_lib.SIGNATURES) == syms


def test_library_exports_every_header_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True)
    exported = set(re.findall(r"\bT (cham_\w+)", out.stdout))
    assert set(header_symbols()) == exported  # nothing missing, nothing extra
    for s in header_symbols():
        assert getattr(lib, s) is not None


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}


def test_limits(lib):
    lim = _lib.limits()
    assert lim.max_rank == 256 and lim.rows_per_page == 8 and lim.max_jobs >= 4
    assert lim.max_segments >= 256 and lim.max_requests >= 4096


def test_errors_are_status_codes(lib):
    pool = ctypes.c_void_p()
    h = _lib.int_array([4096])
    rc = lib.cham_pool_create(ctypes.byref(pool), 0, 4, 1, 1, h, h, 1, 4, 64)
    import torch

    if not torch.cuda.is_available():
        assert rc < 0 and lib.cham_last_error()
    elif rc == 0:
        lib.cham_pool_destroy(pool)
    assert lib.cham_get_limits(None) == -1
    assert lib.cham_lora_apply(None, 0, 0, None, None, 0, None, None, None, None, 0, None, None, None) == -1
    with pytest.raises(_lib.ChamError):
        _lib.call("cham_get_limits", None)


def _pack(dtype, rank, n_layers, h_in, h_out, seed=0):
    rng = np.random.default_rng(seed)
    P = len(h_in)
    a_list, b_list = [], []
    for _l in range(n_layers):
        for p in range(P):
            a = rng.standard_normal((h_in[p], rank)).astype(np.float32)
            b = rng.standard_normal((rank, h_out[p])).astype(np.float32)
            if dtype == _lib.CHAM_BF16:
                a, b = bf16_bits(bf16_round(a)), bf16_bits(bf16_round(b))
            a_list.append(a)
            b_list.append(b)
    es = 4 if dtype == _lib.CHAM_F32 else 2
    page_bytes, _ = geometry(n_layers, h_in, h_out, es)
    n_pages = -(-rank // 8)
    out = np.empty(n_pages * page_bytes, dtype=np.uint8)
    a_flat = np.concatenate([x.reshape(-1) for x in a_list])
    b_flat = np.concatenate([x.reshape(-1) for x in b_list])
    _lib.call("cham_pack_adapter_host_geom", n_layers, P, _lib.int_array(h_in), _lib.int_array(h_out), dtype, rank,
              a_flat.ctypes.data, b_flat.ctypes.data, out.ctypes.data)
    return out, a_list, b_list, es, page_bytes


@pytest.mark.parametrize("dtype,rank,h_in,h_out", [
    (_lib.CHAM_F32, 8, [64, 32], [32, 96]),
    (_lib.CHAM_F32, 20, [128], [64]),
    (_lib.CHAM_BF16, 16, [128, 64, 64], [64, 128, 192]),
    (_lib.CHAM_BF16, 40, [256, 128], [128, 64]),
    (_lib.CHAM_BF16, 1, [64], [64]),
])
def test_host_packing_matches_layout_oracle(lib, dtype, rank, h_in, h_out):
    n_layers = 2
    out, a_list, b_list, es, page_bytes = _pack(dtype, rank, n_layers, h_in, h_out)
    want = pack_adapter(a_list, b_list, rank, n_layers, h_in, h_out, es)
    assert out.tobytes() == want.tobytes()
    # and the layout round-trips: page g holds rank rows 8g..8g+7 of A^T and B
    _, offs = geometry(n_layers, h_in, h_out, es)
    P = len(h_in)
    dt = np.float32 if es == 4 else np.uint16
    for lp, (aoff, boff) in enumerate(offs):
        p = lp % P
        for g in range(-(-rank // 8)):
            page = out[g * page_bytes:(g + 1) * page_bytes]
            at = unpack_block(page, aoff, h_in[p], es, dt)
            bb = unpack_block(page, boff, h_out[p], es, dt)
            rows = slice(8 * g, min(rank, 8 * g + 8))
            n = rows.stop - rows.start
            assert np.array_equal(at[:n], a_list[lp].T[rows]) and not at[n:].any()
            assert np.array_equal(bb[:n], b_list[lp][rows]) and not bb[n:].any()


def test_packing_rejects_bad_geometry(lib):
    h = _lib.int_array([100])
    z = np.zeros(1 << 16, dtype=np.uint8)
    assert lib.cham_pack_adapter_host_geom(1, 1, h, h, 1, 8, z.ctypes.data, z.ctypes.data, z.ctypes.data) == -1
    h = _lib.int_array([64])
    assert lib.cham_pack_adapter_host_geom(1, 1, h, h, 1, 257, z.ctypes.data, z.ctypes.data, z.ctypes.data) == -4
    assert lib.cham_pack_adapter_host_geom(1, 1, h, h, 7, 8, z.ctypes.data, z.ctypes.data, z.ctypes.data) == -1


def test_byte_model_equals_page_geometry():
    """The reference byte model (model.py:23-26: 2,097,152 B per rank unit) is the pool's
    physical size for 7B dims: 8 rank rows x 32 layers x 4 proj x (4096+4096) x 2 B."""
    page_bytes, _ = geometry(32, [4096] * 4, [4096] * 4, 2)
    assert page_bytes == 8 * 2_097_152
