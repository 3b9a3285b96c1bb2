"""All-pairs commutation bitmatrix of a sum (K5).

Row r, bit c of the result is the symplectic-product parity of terms r and c
(1 = anti-commute), restating the all-pairs block of
``group_greedy_parallel`` (grouping.py:136-140) for a whole sum.  Rows are
packed 32 columns per uint32 word, little-endian bit order within the word.
"""

from __future__ import annotations

import torch

from . import _native
from ._device import plane_ld, ptr, stream_ptr
from .sums import PauliSumSoA, _compute_device

METHODS = {"auto": 0, "lists": 1, "direct": 2, "tensor": 3}


def words_per_row(cols: int) -> int:
    return (int(cols) + 31) // 32


def commutation_bitmatrix(s: PauliSumSoA, *, row0: int = 0, rows: int | None = None,
                          col0: int = 0, cols: int | None = None, method: str = "auto",
                          out: torch.Tensor | None = None) -> torch.Tensor:
    """(rows, ceil(cols/32)) uint32 anti-commutation bits for a row block.

    ``col0`` must be a multiple of 32.  The result lives on the compute device
    (a host sum is uploaded; the bits stay on the GPU — use ``.cpu()``).
    """
    dev, _ = _compute_device(s)
    S = s.to(dev).planes()
    M = S.M
    rows = M - row0 if rows is None else int(rows)
    cols = M - col0 if cols is None else int(cols)
    if row0 < 0 or rows < 0 or row0 + rows > M or col0 < 0 or cols < 0 or col0 + cols > M:
        raise IndexError("row/column block out of range")
    if col0 % 32:
        raise ValueError("col0 must be a multiple of 32")
    nw = words_per_row(cols)
    if out is None:
        out = torch.empty((rows, max(nw, 1)), dtype=torch.int32, device=dev)
    ws_bytes = int(_native.load().pl_bitmatrix_workspace_bytes(S.W, rows))
    if method == "lists":  # worst case: every key bit of every row set
        ws_bytes += rows * (128 * S.W + 4 - 64) * 4
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _native.call("pl_commutation_bitmatrix", S.W, M, ptr(S.x), ptr(S.z), S.ld, row0, rows,
                     col0, cols, ptr(out), out.stride(0), METHODS[method], ptr(ws), ws.numel(),
                     stream_ptr(dev))
    return out


def unpack_bits(words: torch.Tensor, cols: int) -> torch.Tensor:
    """(rows, nw) uint32/int32 words -> (rows, cols) uint8 0/1 matrix (host helper)."""
    w = words.to(torch.int64) & 0xFFFFFFFF
    shifts = torch.arange(32, device=w.device, dtype=torch.int64)
    bits = (w.unsqueeze(-1) >> shifts) & 1
    return bits.reshape(w.shape[0], -1)[:, :cols].to(torch.uint8)
