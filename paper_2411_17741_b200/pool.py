"""Paged adapter pool in HBM (Python handle over the C ABI).

Storage side of the reference's adapter cache: `AdapterCache.begin_load` /
`finish_load` (adapter_cache.py:144-159) and the host->GPU link `LinkState.enqueue`
(engine.py:115-121) become page reservation + a pinned `cudaMemcpyAsync` on a side stream
with a completion event.  Decisions (which adapter is resident, which is evicted) stay in
`adapter_cache.AdapterCache`, bit-exact with the reference.

Page geometry (include/chameleon_lora.h): one page = 8 rank rows of one adapter for every
(layer, projection); for Llama-2-7B q/k/v/o in bf16 a page is 16 MiB, i.e. 2 MiB per rank
unit — exactly the reference's byte model DEFAULT_BYTES_PER_RANK_UNIT (model.py:23-26).
"""
from __future__ import annotations

import ctypes
from ctypes import c_size_t, c_void_p

import torch

from . import _lib
from ._lib import CHAM_BF16, CHAM_F32, call

ROWS_PER_PAGE = 8

_TORCH_DTYPE = {CHAM_F32: torch.float32, CHAM_BF16: torch.bfloat16}


def pages_for_rank(rank: int) -> int:
    return -(-int(rank) // ROWS_PER_PAGE)


class AdapterPool:
    """Device pool of `n_pages` pages plus the slot table.

    The caller (PagedAdapterCache) owns page allocation and binds slots with `set_slot`.
    """

    def __init__(self, n_pages: int, n_layers: int, h_in, h_out, dtype=torch.bfloat16,
                 n_slots: int = 1024, max_tokens: int = 8192, device=None):
        if dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("pool dtype must be torch.float32 or torch.bfloat16")
        self.dtype = dtype
        self.cdtype = CHAM_F32 if dtype == torch.float32 else CHAM_BF16
        self.device = torch.device(device if device is not None else "cuda", )
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.n_pages = int(n_pages)
        self.n_layers = int(n_layers)
        self.h_in = [int(h) for h in h_in]
        self.h_out = [int(h) for h in h_out]
        if len(self.h_in) != len(self.h_out):
            raise ValueError("h_in and h_out need one entry per projection")
        self.n_proj = len(self.h_in)
        self.n_slots = int(n_slots)
        self.max_tokens = int(max_tokens)
        handle = c_void_p()
        call("cham_pool_create", ctypes.byref(handle), self.device.index, self.n_pages, self.n_layers,
             self.n_proj, _lib.int_array(self.h_in), _lib.int_array(self.h_out), self.cdtype,
             self.n_slots, self.max_tokens)
        self._h = handle
        pb = c_size_t()
        call("cham_pool_page_bytes", self._h, ctypes.byref(pb))
        self.page_bytes = int(pb.value)
        self.slot_rank = [0] * self.n_slots
        self.slot_pages: list[list[int]] = [[] for _ in range(self.n_slots)]

    # -- lifecycle ---------------------------------------------------------------------
    @property
    def handle(self) -> c_void_p:
        if self._h is None:
            raise RuntimeError("pool already destroyed")
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            _lib.lib().cham_pool_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    # -- geometry ----------------------------------------------------------------------
    @property
    def elem_bytes(self) -> int:
        return 4 if self.cdtype == CHAM_F32 else 2

    def block_offsets(self, layer: int, proj: int) -> tuple[int, int]:
        a, b = c_size_t(), c_size_t()
        call("cham_pool_block_offsets", self.handle, layer, proj, ctypes.byref(a), ctypes.byref(b))
        return int(a.value), int(b.value)

    def base_ptr(self) -> int:
        out = c_void_p()
        call("cham_pool_base", self.handle, ctypes.byref(out))
        return int(out.value or 0)

    def adapter_bytes(self, rank: int) -> int:
        return pages_for_rank(rank) * self.page_bytes

    # -- slot table --------------------------------------------------------------------
    def set_slot(self, slot: int, rank: int, pages, stream=None) -> None:
        pages = [int(p) for p in pages]
        call("cham_pool_set_slot", self.handle, int(slot), int(rank), _lib.int_array(pages), len(pages),
             _stream_ptr(stream))
        self.slot_rank[slot] = int(rank)
        self.slot_pages[slot] = pages

    # -- cross-apply weight prefetch ----------------------------------------------------
    def set_next_apply(self, layer: int = -1, projs=()) -> None:
        """Hint: the apply launched after the next one is (layer, projs) on the same plan
        (cham_pool_set_next_apply; consumed by the next apply).  Empty projs clears it."""
        projs = [int(p) for p in projs]
        call("cham_pool_set_next_apply", self.handle, int(layer), len(projs), _lib.int_array(projs) if projs else None)

    def set_l2_prefetch(self, nbytes: int) -> None:
        """Budget of hinted A-block bytes an apply pulls into L2 once out of units (0 = off)."""
        call("cham_pool_set_l2_prefetch", self.handle, int(nbytes))

    # -- device errors -----------------------------------------------------------------
    def device_error(self, clear: bool = True, stream=None) -> int:
        """The kernels' device-side error word (0 = none); synchronises the stream."""
        v = ctypes.c_int()
        call("cham_pool_device_error", self.handle, ctypes.byref(v), 1 if clear else 0, _stream_ptr(stream))
        return int(v.value)

    def check_device_error(self, stream=None) -> None:
        """Raise ChamError if a kernel hit a device-side limit (its apply left y untouched)."""
        v = self.device_error(clear=True, stream=stream)
        if v:
            raise _lib.ChamError(v, "device kernel", "a launch met a compiled-in limit on the device "
                                 "(segments, prefill tiles or plan tokens) and skipped its work")

    # -- routing -----------------------------------------------------------------------
    def set_prefill_route(self, min_tokens: int = 64, min_segment_tokens: int = 0,
                          max_segment_tokens: int = -1) -> None:
        """Segments with >= min_tokens tokens (rank <= 128) run on the tcgen05 prefill kernels
        (bf16 pools only); min_tokens <= 0 sends everything to the decode kernel.  The
        segment-length hints (0 / -1 = unknown) let a launch skip the kernel family that has
        no work; set them before the step's plan is built."""
        call("cham_pool_set_prefill_route", self.handle, int(min_tokens), int(min_segment_tokens),
             int(max_segment_tokens))

    # -- packing -----------------------------------------------------------------------
    def _flatten(self, a_list, b_list, rank: int, device):
        n_lp = self.n_layers * self.n_proj
        if len(a_list) != n_lp or len(b_list) != n_lp:
            raise ValueError(f"need {n_lp} A and B matrices (layers x projections)")
        flat_a, flat_b = [], []
        for lp in range(n_lp):
            p = lp % self.n_proj
            a, b = a_list[lp], b_list[lp]
            if tuple(a.shape) != (self.h_in[p], rank) or tuple(b.shape) != (rank, self.h_out[p]):
                raise ValueError(f"(l,p)={divmod(lp, self.n_proj)}: A must be [{self.h_in[p]}, {rank}] and "
                                 f"B [{rank}, {self.h_out[p]}]")
            flat_a.append(a.to(device=device, dtype=self.dtype).contiguous().reshape(-1))
            flat_b.append(b.to(device=device, dtype=self.dtype).contiguous().reshape(-1))
        return torch.cat(flat_a), torch.cat(flat_b)

    def pack_host(self, a_list, b_list, rank: int, pin: bool = True) -> torch.Tensor:
        """Pack one adapter (A [h_in, r], B [r, h_out] per (layer, proj)) into page format in
        (pinned) host memory, ready for `fill_async`."""
        fa, fb = self._flatten(a_list, b_list, rank, "cpu")
        out = torch.empty(self.adapter_bytes(rank), dtype=torch.uint8, pin_memory=pin)
        call("cham_pack_adapter_host", self.handle, int(rank), fa.data_ptr(), fb.data_ptr(), out.data_ptr())
        return out

    def pack_device(self, a_list, b_list, rank: int, stream=None) -> torch.Tensor:
        fa, fb = self._flatten(a_list, b_list, rank, self.device)
        out = torch.empty(self.adapter_bytes(rank), dtype=torch.uint8, device=self.device)
        call("cham_pack_adapter_device", self.handle, int(rank), fa.data_ptr(), fb.data_ptr(), out.data_ptr(),
             _stream_ptr(stream))
        return out

    # -- fills -------------------------------------------------------------------------
    def fill_async(self, slot: int, packed_host: torch.Tensor, stream=None, event=None) -> None:
        """Pinned host -> HBM copy of a packed adapter into the slot's pages on `stream`
        (the side stream of the miss path); `event` (torch.cuda.Event) is recorded after."""
        if packed_host.device.type != "cpu":
            raise ValueError("fill_async takes a host tensor (use fill_from_device for device data)")
        call("cham_pool_fill_async", self.handle, int(slot), packed_host.data_ptr(), packed_host.numel(),
             _stream_ptr(stream), None)
        if event is not None:
            event.record(stream if stream is not None else torch.cuda.current_stream(self.device))

    def fill_from_device(self, slot: int, packed_dev: torch.Tensor, stream=None) -> None:
        call("cham_pool_fill_from_device", self.handle, int(slot), packed_dev.data_ptr(), packed_dev.numel(),
             _stream_ptr(stream))

    def read_page(self, page: int, stream=None) -> torch.Tensor:
        """Copy one page back to the host (uint8) — introspection / tests."""
        out = torch.empty(self.page_bytes, dtype=torch.uint8)
        call("cham_pool_copy_out", self.handle, int(page) * self.page_bytes, self.page_bytes, out.data_ptr(),
             _stream_ptr(stream))
        return out


def _stream_ptr(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream
