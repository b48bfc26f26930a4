"""ctypes binding of the in-tree C-ABI extension `libchameleon_lora.so`.

The product path has no CPU fallback: if the shared library is missing or a call fails,
a `ChamError` is raised.  Every symbol declared in include/chameleon_lora.h is bound here
(tests/test_abi.py checks the two lists agree).
"""
from __future__ import annotations

import ctypes
from ctypes import POINTER, c_int, c_size_t, c_void_p, c_char_p
from pathlib import Path

import os

# CHAM_LIB overrides the in-tree library (used for A/B builds in experiments only)
LIB_PATH = Path(os.environ.get("CHAM_LIB") or Path(__file__).resolve().with_name("libchameleon_lora.so"))

CHAM_F32 = 0
CHAM_BF16 = 1


class ChamError(RuntimeError):
    """A C-ABI call returned a negative cham_status."""

    def __init__(self, code: int, what: str, msg: str):
        super().__init__(f"{what} failed (status {code}): {msg}")
        self.code = code


class ChamLimits(ctypes.Structure):
    _fields_ = [
        ("max_rank", c_int),
        ("max_segments", c_int),
        ("max_jobs", c_int),
        ("max_requests", c_int),
        ("rows_per_page", c_int),
        ("tokens_per_tile", c_int),
        ("prefill_min_tokens", c_int),
    ]


_P = c_void_p
_IP = POINTER(c_int)
SIGNATURES = {
    "cham_last_error": (c_char_p, []),
    "cham_get_limits": (c_int, [POINTER(ChamLimits)]),
    "cham_device_sm_count": (c_int, [c_int, _IP]),
    "cham_pool_create": (c_int, [POINTER(_P), c_int, c_int, c_int, c_int, _IP, _IP, c_int, c_int, c_int]),
    "cham_pool_destroy": (c_int, [_P]),
    "cham_pool_page_bytes": (c_int, [_P, POINTER(c_size_t)]),
    "cham_pool_block_offsets": (c_int, [_P, c_int, c_int, POINTER(c_size_t), POINTER(c_size_t)]),
    "cham_pool_base": (c_int, [_P, POINTER(_P)]),
    "cham_pool_set_slot": (c_int, [_P, c_int, c_int, _IP, c_int, _P]),
    "cham_pool_fill_async": (c_int, [_P, c_int, _P, c_size_t, _P, _P]),
    "cham_pool_fill_from_device": (c_int, [_P, c_int, _P, c_size_t, _P]),
    "cham_pool_set_prefill_route": (c_int, [_P, c_int, c_int, c_int]),
    "cham_pool_device_error": (c_int, [_P, _IP, c_int, _P]),
    "cham_pool_set_next_apply": (c_int, [_P, c_int, c_int, _IP]),
    "cham_pool_set_l2_prefetch": (c_int, [_P, ctypes.c_longlong]),
    "cham_debug_set_trace": (c_int, [_P, _P, c_int]),
    "cham_pool_copy_out": (c_int, [_P, c_size_t, c_size_t, _P, _P]),
    "cham_pack_adapter_host": (c_int, [_P, c_int, _P, _P, _P]),
    "cham_pack_adapter_host_geom": (c_int, [c_int, c_int, _IP, _IP, c_int, c_int, _P, _P, _P]),
    "cham_pack_adapter_device": (c_int, [_P, c_int, _P, _P, _P, _P]),
    "cham_build_segments": (c_int, [_P, _P, _P, c_int, _P, _P, _P, _P, _P, _P]),
    "cham_plan_bytes": (c_size_t, [_P]),
    "cham_build_plan": (c_int, [_P, _P, _P, _P, _P, c_int, _P, _P, _P]),
    "cham_lora_apply": (c_int, [_P, c_int, c_int, _P, _P, c_int, _P, _P, _P, _P, c_int, _P, _P, _P]),
    "cham_lora_apply_multi": (c_int, [_P, c_int, c_int, _IP, POINTER(_P), POINTER(_P), c_int, _P, _P, _P, _P,
                                      c_int, _P, _P, _P]),
    "cham_lora_shrink": (c_int, [_P, c_int, c_int, _P, _P, c_int, c_int, _P, _P, _P, _P, c_int, _P, _P, _P]),
    "cham_lora_expand": (c_int, [_P, c_int, c_int, _P, c_int, _P, c_int, _P, _P, _P, _P, c_int, _P, _P, _P]),
    "cham_lora_shrink_multi": (c_int, [_P, c_int, c_int, _P, _P, _P, c_int, c_int, c_int, _P, _P, _P, _P, c_int, _P,
                                       _P, _P]),
    "cham_lora_expand_multi": (c_int, [_P, c_int, c_int, _P, _P, c_int, c_int, _P, c_int, _P, _P, _P, _P, c_int, _P,
                                       _P, _P]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load the extension once; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ChamError(-5, "load", f"{LIB_PATH} is missing — build it with "
                                        "`python -c 'import __graft_entry__ as g; g.build()'`")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().cham_last_error()
        raise ChamError(rc, what, msg.decode() if msg else "")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def limits() -> ChamLimits:
    out = ChamLimits()
    call("cham_get_limits", ctypes.byref(out))
    return out


def ptr(t) -> int | None:
    """Raw device/host pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def int_array(values) -> ctypes.Array:
    arr = (c_int * len(values))(*[int(v) for v in values])
    return arr
