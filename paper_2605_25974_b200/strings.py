"""Bit-packed Pauli strings with exact 2-bit phase tracking (host value type).

Mirrors ``paulialg/strings.py``: a string is i^k times a tensor product of
letters encoded per qubit as (x, z): I=(0,0), X=(1,0), Z=(0,1), Y=(1,1)
(strings.py:3-6); values are immutable (strings.py:90-91).  Label parsing,
formatting and the canonical key are host bookkeeping; the algebra
(``multiply``, ``product_phase_exponent``, ``symplectic_inner_product``) runs on
the GPU through the batched kernels of the C ABI (a batch of one pair), the
same kernels the sum-level paths use.  Batched device entry points
(:func:`batch_multiply`, :func:`batch_sip`) take (W, P) planes directly.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import _native
from ._device import cuda_device, i64_tensor_to_u64, plane_ld, ptr, stream_ptr, u64_to_i64_tensor
from .bits import (DimensionError, PHASE_FACTORS, check_padding, format_label, parse_label,
                   tier_for, words_for)


class PauliString:
    """Fixed-capacity n-qubit Pauli operator with global phase i^k (strings.py:54-184)."""

    __slots__ = ("n", "tier", "x", "z", "phase")

    def __init__(self, n: int, x_words, z_words, phase: int = 0, *, validate: bool = True):
        self.n = int(n)
        self.tier = tier_for(self.n)
        x = np.array(x_words, dtype=np.uint64, copy=True).reshape(-1)
        z = np.array(z_words, dtype=np.uint64, copy=True).reshape(-1)
        if validate:
            W = self.tier // 64
            if x.shape != (W,) or z.shape != (W,):
                raise ValueError(f"expected {W} words per vector for {self.n} qubits, got shapes "
                                 f"{x.shape} and {z.shape}")
            if not check_padding(x, z, self.n):
                raise ValueError("nonzero padding bits at positions >= n")
        x.flags.writeable = False
        z.flags.writeable = False
        self.x, self.z = x, z
        self.phase = int(phase) % 4

    @classmethod
    def from_label(cls, label: str, phase: int = 0) -> "PauliString":
        x, z, n = parse_label(label)
        return cls(n, x, z, phase, validate=False)

    @classmethod
    def identity(cls, n: int) -> "PauliString":
        W = words_for(n)
        return cls(n, np.zeros(W, np.uint64), np.zeros(W, np.uint64), 0, validate=False)

    def to_label(self) -> tuple[str, int]:
        return format_label(self.x, self.z, self.n), self.phase

    @property
    def label(self) -> str:
        return format_label(self.x, self.z, self.n)

    @property
    def phase_factor(self) -> complex:
        return complex(PHASE_FACTORS[self.phase])

    @property
    def words(self) -> int:
        return self.tier // 64

    def _check_same_n(self, other: "PauliString") -> None:
        if self.n != other.n:
            raise DimensionError(f"qubit counts differ: {self.n} != {other.n}")

    def product_phase_exponent(self, other: "PauliString") -> int:
        """Letter-product phase, flags excluded (strings.py:128-131)."""
        self._check_same_n(other)
        _, _, k = _pair_multiply(self.x, self.z, 0, other.x, other.z, 0)
        return k

    def multiply(self, other: "PauliString") -> "PauliString":
        """Exact product, left operand self (strings.py:133-137)."""
        self._check_same_n(other)
        x, z, k = _pair_multiply(self.x, self.z, self.phase, other.x, other.z, other.phase)
        return PauliString(self.n, x, z, k, validate=False)

    __mul__ = multiply

    def symplectic_inner_product(self, other: "PauliString") -> int:
        """0 when the strings commute, 1 when they anti-commute (strings.py:141-144)."""
        self._check_same_n(other)
        return _pair_sip(self.x, self.z, other.x, other.z)

    def commutes(self, other: "PauliString") -> bool:
        return self.symplectic_inner_product(other) == 0

    def weight(self) -> int:
        return int(np.bitwise_count(self.x | self.z).sum())

    def apply_clifford(self, gate: str, qubits) -> "PauliString":
        """U * self * U^dagger for a Clifford gate (strings.py:153-163); a new
        string.  Runs the f2 kernel (``pl_apply_clifford``) on a one-term sum."""
        from . import gates

        if isinstance(qubits, (int, np.integer)):
            qubits = (int(qubits),)
        else:
            qubits = tuple(int(q) for q in qubits)
        code, q0, q1 = gates.check_gate(gate, qubits, self.n)
        dev = cuda_device()
        x = _dev_planes(self.x, dev)
        z = _dev_planes(self.z, dev)
        k = torch.tensor([self.phase], dtype=torch.uint8, device=dev)
        with torch.cuda.device(dev):
            gates.apply_clifford_planes(x, z, k, 1, self.words, 1, code, q0, q1, dev)
        return PauliString(self.n, i64_tensor_to_u64(x)[:, 0], i64_tensor_to_u64(z)[:, 0],
                           int(k.item()), validate=False)

    def canonical_key(self) -> bytes:
        """(z words, x words) big-endian, phase ignored (strings.py:165-167)."""
        return self.z.astype(">u8").tobytes() + self.x.astype(">u8").tobytes()

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, PauliString):
            return NotImplemented
        return (self.n == other.n and self.phase == other.phase
                and bool(np.array_equal(self.x, other.x)) and bool(np.array_equal(self.z, other.z)))

    def __hash__(self) -> int:
        return hash((self.n, self.phase, self.x.tobytes(), self.z.tobytes()))

    def __repr__(self) -> str:
        return f"PauliString({('', 'i*', '-', '-i*')[self.phase]}{self.label})"


# --------------------------------------------------------- device kernels
def _dev_planes(words: np.ndarray, dev) -> torch.Tensor:
    return u64_to_i64_tensor(np.ascontiguousarray(words.reshape(-1, 1))).to(dev)


def _host_words(v) -> np.ndarray:
    return np.ascontiguousarray(v, dtype=np.uint64)


def _pair_host(ax, az, ak, bx, bz, bk, want_product: bool):
    """One launch of ``pl_pair_host``: (x, z, k) of a*b, or the anti-commutation bit."""
    import ctypes as C

    dev = cuda_device()
    ax, az, bx, bz = (_host_words(v) for v in (ax, az, bx, bz))
    W = ax.shape[0]
    with torch.cuda.device(dev):
        if want_product:
            ox, oz = np.empty(W, np.uint64), np.empty(W, np.uint64)
            ok = C.c_int(0)
            _native.call("pl_pair_host", W, ax.ctypes.data, az.ctypes.data, int(ak),
                         bx.ctypes.data, bz.ctypes.data, int(bk), ox.ctypes.data, oz.ctypes.data,
                         C.addressof(ok), None, stream_ptr(dev))
            return ox, oz, int(ok.value)
        anti = C.c_int(0)
        _native.call("pl_pair_host", W, ax.ctypes.data, az.ctypes.data, 0, bx.ctypes.data,
                     bz.ctypes.data, 0, None, None, None, C.addressof(anti), stream_ptr(dev))
        return int(anti.value)


def _pair_multiply(ax, az, ak, bx, bz, bk):
    return _pair_host(ax, az, ak, bx, bz, bk, True)


def _pair_sip(ax, az, bx, bz) -> int:
    return _pair_host(ax, az, 0, bx, bz, 0, False)


def batch_multiply(ax, az, ak, bx, bz, bk):
    """Batched pair multiply on (W, P) device planes (bench.py:168-177 over SoA).

    Returns (x, z, k) as new device tensors: (W, P) int64 planes holding the
    uint64 words and (P,) uint8 phase exponents.  ``ak``/``bk`` may be None.
    """
    W, P = ax.shape
    dev = ax.device
    if dev.type != "cuda":
        raise _native.NativeLibraryError("batch_multiply needs CUDA tensors")
    ox = torch.empty((W, P), dtype=torch.int64, device=dev)
    oz = torch.empty((W, P), dtype=torch.int64, device=dev)
    ok = torch.empty(P, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _native.call("pl_batch_multiply", W, P, ptr(ax), ptr(az), ptr(ak), plane_ld(ax),
                     ptr(bx), ptr(bz), ptr(bk), plane_ld(bx), ptr(ox), ptr(oz), ptr(ok), P,
                     stream_ptr(dev))
    return ox, oz, ok


def batch_sip(ax, az, bx, bz):
    """Per-pair anti-commutation bit (strings.py:47-51) on (W, P) device planes."""
    W, P = ax.shape
    dev = ax.device
    out = torch.empty(P, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _native.call("pl_batch_sip", W, P, ptr(ax), ptr(az), plane_ld(ax), ptr(bx), ptr(bz),
                     plane_ld(bx), ptr(out), stream_ptr(dev))
    return out


def batch_pair_multiply(ax, az, aflags, bx, bz, bflags):
    """Drop-in for the reference's ``_batch_pair_multiply`` (bench.py:168-177).

    Accepts the reference's host (P, W) uint64 columns + (P,) flags and returns
    host (x, z, k) in the same layout; the work runs on the GPU (upload,
    kernel, download).  Device (W, P) tensors go through :func:`batch_multiply`.
    """
    if isinstance(ax, torch.Tensor) and ax.device.type == "cuda":
        return batch_multiply(ax, az, aflags, bx, bz, bflags)
    dev = cuda_device()
    planes = [u64_to_i64_tensor(np.ascontiguousarray(np.asarray(v, dtype=np.uint64).T)).to(dev)
              for v in (ax, az, bx, bz)]
    fa = torch.from_numpy(np.ascontiguousarray(aflags, dtype=np.uint8)).to(dev)
    fb = torch.from_numpy(np.ascontiguousarray(bflags, dtype=np.uint8)).to(dev)
    x, z, k = batch_multiply(planes[0], planes[1], fa, planes[2], planes[3], fb)
    return (np.ascontiguousarray(i64_tensor_to_u64(x).T), np.ascontiguousarray(i64_tensor_to_u64(z).T),
            k.cpu().numpy())


# ------------------------------------------------------ module functions
def ps_from_label(label: str, phase: int = 0) -> PauliString:
    return PauliString.from_label(label, phase)


def ps_to_label(p: PauliString) -> tuple[str, int]:
    return p.to_label()


def product_phase_exponent(a: PauliString, b: PauliString) -> int:
    return a.product_phase_exponent(b)


def ps_multiply(a: PauliString, b: PauliString) -> PauliString:
    return a.multiply(b)


def symplectic_inner_product(a: PauliString, b: PauliString) -> int:
    return a.symplectic_inner_product(b)


def ps_commutes(a: PauliString, b: PauliString) -> bool:
    return a.commutes(b)


def ps_weight(p: PauliString) -> int:
    return p.weight()


def ps_apply_clifford(p: PauliString, gate: str, qubits) -> PauliString:
    """strings.py:215-216."""
    return p.apply_clifford(gate, qubits)
