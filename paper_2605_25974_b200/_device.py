"""Device plumbing: torch tensors as plain device buffers for the C ABI.

PyTorch supplies device memory, streams and host<->device copies; all Pauli
arithmetic happens in the native kernels.  uint64 bit planes are stored as
torch.int64 (same bits) because torch's uint64 op coverage is partial.
"""

from __future__ import annotations

import numpy as np
import torch

from ._native import NativeLibraryError


def cuda_device(device=None) -> torch.device:
    """Resolve the CUDA device to compute on; fail loudly without a GPU."""
    if device is not None:
        d = torch.device(device)
        if d.type == "cuda":
            return d
    if not torch.cuda.is_available():
        raise NativeLibraryError(
            "paulib_b200 computes on CUDA only (no CPU fallback) and no GPU is visible")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t):
    """Device (or host) address of a tensor, or None."""
    if t is None:
        return None
    return t.data_ptr() if t.numel() else None


def u64_to_i64_tensor(a) -> torch.Tensor:
    """numpy uint64 / torch int64|uint64 -> torch int64 with the same bits."""
    if isinstance(a, torch.Tensor):
        if a.dtype == torch.int64:
            return a
        if a.dtype == torch.uint64:
            return a.view(torch.int64)
        raise TypeError(f"bit planes must be 64-bit integer tensors, got {a.dtype}")
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    # torch needs writable memory (PauliString's planes are read-only) and
    # strides in whole elements (a one-record field view of packed AoS records
    # is "contiguous" with the record's odd stride)
    if not arr.flags.writeable or any(st % arr.itemsize for st in arr.strides):
        arr = arr.copy()
    return torch.from_numpy(arr.view(np.int64))


def i64_tensor_to_u64(t: torch.Tensor) -> np.ndarray:
    """torch int64 planes -> numpy uint64 (copies to host if needed)."""
    return t.detach().cpu().contiguous().numpy().view(np.uint64)


def as_u8(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(torch.uint8)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.uint8)))


def as_c128(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(torch.complex128)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.complex128)))


def plane_ld(t: torch.Tensor) -> int:
    """Leading dimension (words between planes) of a (W, M) plane tensor."""
    if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1):
        raise ValueError("bit planes must be (W, M) with unit stride along M")
    return max(t.stride(0), t.shape[1], 1)


def c128_ptr(t: torch.Tensor):
    return ptr(t)
