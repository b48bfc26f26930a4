"""Numpy restatement of the paged adapter-pool layout (test infrastructure only).

Page = 8 rank rows of one adapter for every (layer, projection).  Per (l, p) block: A^T
[8, h_in] then B [8, h_out], each tiled in 1 KiB atoms (8 rows x 128 bytes) with the
128-byte XOR swizzle: 16-byte chunk c of row j is stored at chunk position c ^ j.
This mirrors include/chameleon_lora.h and is used to check cham_pack_adapter_* and pool
read-back bit-exactly.
"""
from __future__ import annotations

import numpy as np

ROWS = 8
ROW_BYTES = 128
ATOM = 1024


def geometry(n_layers, h_in, h_out, es):
    offs = []
    off = 0
    for _l in range(n_layers):
        for p in range(len(h_in)):
            a = off
            off += ROWS * h_in[p] * es
            b = off
            off += ROWS * h_out[p] * es
            offs.append((a, b))
    return off, offs


def _tile(mat_rows: np.ndarray, es: int) -> np.ndarray:
    """mat_rows: [8, n] of element size es (as uint8 view [8, n*es]) -> swizzled atoms bytes."""
    rows, nbytes = mat_rows.shape
    assert rows == ROWS and nbytes % ROW_BYTES == 0
    n_atoms = nbytes // ROW_BYTES
    # [8, n_atoms, 8 chunks, 16] -> [n_atoms, 8 rows, 8 chunks, 16]
    t = mat_rows.reshape(ROWS, n_atoms, 8, 16).transpose(1, 0, 2, 3).copy()
    out = np.empty_like(t)
    for j in range(ROWS):
        for c in range(8):
            out[:, j, c ^ j, :] = t[:, j, c, :]
    return out.reshape(-1)


def pack_adapter(a_list, b_list, rank, n_layers, h_in, h_out, es):
    """a_list[l*P+p]: [h_in, rank]; b_list[l*P+p]: [rank, h_out] (numpy arrays whose itemsize
    is es).  Returns uint8 [ceil(rank/8) * page_bytes]."""
    page_bytes, offs = geometry(n_layers, h_in, h_out, es)
    np_ = -(-rank // ROWS)
    out = np.zeros(np_ * page_bytes, dtype=np.uint8)
    P = len(h_in)
    for lp, (aoff, boff) in enumerate(offs):
        p = lp % P
        a = np.ascontiguousarray(a_list[lp])
        b = np.ascontiguousarray(b_list[lp])
        at = np.zeros((np_ * ROWS, h_in[p]), dtype=a.dtype)
        at[:rank] = a.T
        bb = np.zeros((np_ * ROWS, h_out[p]), dtype=b.dtype)
        bb[:rank] = b
        for g in range(np_):
            base = g * page_bytes
            ab = at[g * ROWS:(g + 1) * ROWS].view(np.uint8).reshape(ROWS, -1)
            bbb = bb[g * ROWS:(g + 1) * ROWS].view(np.uint8).reshape(ROWS, -1)
            out[base + aoff: base + aoff + ab.size] = _tile(ab, es)
            out[base + boff: base + boff + bbb.size] = _tile(bbb, es)
    return out


def unpack_block(page_bytes_arr: np.ndarray, off: int, n: int, es: int, dtype) -> np.ndarray:
    """Inverse of _tile for one [8, n] block starting at byte `off` of a page."""
    nbytes = n * es
    n_atoms = nbytes // ROW_BYTES
    t = page_bytes_arr[off: off + ROWS * nbytes].reshape(n_atoms, ROWS, 8, 16)
    out = np.empty_like(t)
    for j in range(ROWS):
        for c in range(8):
            out[:, j, c, :] = t[:, j, c ^ j, :]
    return out.transpose(1, 0, 2, 3).reshape(ROWS, nbytes).copy().view(dtype)
