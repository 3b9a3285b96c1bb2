"""Weighted Pauli sums: device-resident SoA planes (the hot-path storage) and the
reference's packed AoS records, behind the reference's public API.

Mirrors ``paulialg/sums.py``:

* :class:`PauliSumSoA` — the north-star layout (sums.py:429-477): x, z as
  (W, M) uint64 planes, a phase byte and a complex128 coefficient per term.
  Here the planes are torch tensors, normally on a CUDA device; a sum whose
  tensors live on the host is uploaded for every operation and its results
  come back to the host (the end-to-end path).
* :class:`PauliSum` — the packed array-of-structures record
  ``x[W] u64, z[W] u64, flags u8, coeff c128`` (sums.py:48-57, :360-426),
  kept on the host as a numpy structured array for drop-in compatibility;
  operations transpose it to SoA planes on the device.
* ``multiply`` (sums.py:293-305), ``sort_and_combine`` (sums.py:286-291),
  ``sum_multiply`` / ``sort_and_combine`` module wrappers (sums.py:484-489).

All arithmetic runs in the native CUDA kernels (no CPU fallback).  The
``threads`` argument of ``multiply`` is accepted for signature compatibility;
the GPU result is bit-identical for every value, as the reference guarantees
for its thread split (sums.py:296-299).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Iterable, Iterator, Sequence, Union

import numpy as np
import torch

from . import _native
from ._device import (as_c128, as_u8, cuda_device, i64_tensor_to_u64, plane_ld, ptr, stream_ptr,
                      u64_to_i64_tensor)
from .bits import DimensionError, PHASE_FACTORS, tier_for
from .strings import PauliString


@dataclass(frozen=True)
class PauliTerm:
    """One (coefficient, string) entry of a sum (sums.py:31-42)."""

    coeff: complex
    string: PauliString

    def __post_init__(self):
        c = complex(self.coeff)
        if not (math.isfinite(c.real) and math.isfinite(c.imag)):
            raise ValueError(f"coefficient must be finite, got {c}")
        object.__setattr__(self, "coeff", c)


TermEntry = Union[PauliTerm, tuple]


def aos_dtype(words: int) -> np.dtype:
    """Packed record: x-words, z-words, flags byte, coefficient (sums.py:48-57)."""
    return np.dtype([("x", np.uint64, (words,)), ("z", np.uint64, (words,)),
                     ("flags", np.uint8), ("coeff", np.complex128)])


def _entries_to_columns(entries: Sequence[TermEntry], n: int | None):
    """(coeff, label-or-string) entries -> (n, x (M,W), z, flags, coeffs) (sums.py:60-91)."""
    coeffs, strings = [], []
    for e in entries:
        c, s = (e.coeff, e.string) if isinstance(e, PauliTerm) else e
        if not isinstance(s, PauliString):
            s = PauliString.from_label(str(s))
        c = complex(c)
        if not (math.isfinite(c.real) and math.isfinite(c.imag)):
            raise ValueError(f"coefficient must be finite, got {c}")
        if n is None:
            n = s.n
        elif s.n != n:
            raise DimensionError(f"term on {s.n} qubits in a {n}-qubit sum")
        coeffs.append(c)
        strings.append(s)
    if n is None:
        raise ValueError("qubit count required for an empty sum")
    W = tier_for(n) // 64
    m = len(strings)
    x = np.zeros((m, W), np.uint64)
    z = np.zeros((m, W), np.uint64)
    flags = np.zeros(m, np.uint8)
    for i, s in enumerate(strings):
        x[i], z[i], flags[i] = s.x, s.z, s.phase
    return n, x, z, flags, np.array(coeffs, dtype=np.complex128).reshape(m)


def _check_finite_np(c: np.ndarray) -> None:
    if c.size and not np.isfinite(c).all():
        raise ValueError("coefficients must be finite")


class _Planes:
    """Device view of a sum: (W, M) int64 planes + flags + coeffs on one device."""

    __slots__ = ("x", "z", "k", "c", "W", "M", "ld")

    def __init__(self, x, z, k, c):
        if plane_ld(x) != plane_ld(z):
            x, z = x.contiguous(), z.contiguous()
        self.x, self.z, self.k, self.c = x, z, k.contiguous(), c.contiguous()
        self.W, self.M = x.shape
        self.ld = plane_ld(x)


class PauliSumSoA:
    """Struct-of-arrays sum: word w of every term contiguous (sums.py:429-477).

    ``x``/``z`` are (W, M) torch.int64 tensors holding uint64 bit patterns
    (unit stride along M; the plane stride may exceed M), ``flags`` (M,)
    uint8 and ``coeffs`` (M,) complex128, all on one device.
    """

    __slots__ = ("n", "tier", "x", "z", "flags", "coeffs")

    def __init__(self, n, x, z, flags, coeffs, *, device=None, validate: bool = True):
        self.n = int(n)
        self.tier = tier_for(self.n)
        W = self.tier // 64
        if validate and not isinstance(coeffs, torch.Tensor):
            _check_finite_np(np.asarray(coeffs, dtype=np.complex128))
        xt, zt = u64_to_i64_tensor(x), u64_to_i64_tensor(z)
        if xt.dim() != 2 or xt.shape[0] != W or zt.shape != xt.shape:
            raise ValueError(f"expected ({W}, M) word arrays, got {tuple(xt.shape)} and "
                             f"{tuple(zt.shape)}")
        m = xt.shape[1]
        ft, ct = as_u8(flags), as_c128(coeffs)
        if ft.shape != (m,) or ct.shape != (m,):
            raise ValueError("flags and coeffs must have one entry per term")
        if device is not None:
            dev = torch.device(device)
            nb = dev.type == "cuda"
            xt, zt = xt.to(dev, non_blocking=nb), zt.to(dev, non_blocking=nb)
            ft, ct = ft.to(dev, non_blocking=nb), ct.to(dev, non_blocking=nb)
        if validate and isinstance(coeffs, torch.Tensor) and ct.numel():
            if not bool(torch.isfinite(torch.view_as_real(ct)).all()):
                raise ValueError("coefficients must be finite")
        self.x, self.z, self.flags, self.coeffs = xt, zt, ft, ct

    # ----------------------------------------------------------- creation
    @classmethod
    def from_columns(cls, n, x, z, flags, coeffs, *, device=None, validate=True):
        """From the reference's (M, W) column layout (sums.py:455-457)."""
        x = np.asarray(x, dtype=np.uint64)
        z = np.asarray(z, dtype=np.uint64)
        W = tier_for(n) // 64
        x = x.reshape(-1, W)
        z = z.reshape(-1, W)
        return cls(n, np.ascontiguousarray(x.T), np.ascontiguousarray(z.T), flags, coeffs,
                   device=device, validate=validate)

    _from_columns = from_columns

    @classmethod
    def from_terms(cls, entries: Iterable[TermEntry], n: int | None = None, *, device=None):
        n, x, z, flags, coeffs = _entries_to_columns(list(entries), n)
        return cls.from_columns(n, x, z, flags, coeffs, device=device)

    @classmethod
    def empty(cls, n: int, device=None):
        W = tier_for(n) // 64
        return cls(n, np.zeros((W, 0), np.uint64), np.zeros((W, 0), np.uint64),
                   np.zeros(0, np.uint8), np.zeros(0, np.complex128), device=device)

    # -------------------------------------------------------------- views
    @property
    def words(self) -> int:
        return self.tier // 64

    @property
    def device(self) -> torch.device:
        return self.x.device

    def __len__(self) -> int:
        return int(self.x.shape[1])

    def to(self, device) -> "PauliSumSoA":
        dev = torch.device(device)
        if dev == self.device:
            return self
        nb = dev.type == "cuda"
        out = object.__new__(PauliSumSoA)
        out.n, out.tier = self.n, self.tier
        out.x = self.x.to(dev, non_blocking=nb)
        out.z = self.z.to(dev, non_blocking=nb)
        out.flags = self.flags.to(dev, non_blocking=nb)
        out.coeffs = self.coeffs.to(dev, non_blocking=nb)
        return out

    def cuda(self, device=None) -> "PauliSumSoA":
        return self.to(cuda_device(device))

    def cpu(self) -> "PauliSumSoA":
        return self.to("cpu")

    def columns(self):
        """Host numpy (x (M,W), z (M,W), flags, coeffs) (sums.py:459-460)."""
        x = i64_tensor_to_u64(self.x).T
        z = i64_tensor_to_u64(self.z).T
        return (x, z, self.flags.detach().cpu().numpy(), self.coeffs.detach().cpu().numpy())

    _columns = columns

    def planes(self) -> _Planes:
        return _Planes(self.x, self.z, self.flags, self.coeffs)

    @property
    def payload_nbytes(self) -> int:
        m = len(self)
        return 2 * self.words * 8 * m + m + 16 * m

    def term(self, i: int) -> PauliTerm:
        x, z = i64_tensor_to_u64(self.x[:, i:i + 1])[:, 0], i64_tensor_to_u64(self.z[:, i:i + 1])[:, 0]
        k = int(self.flags[i].item())
        c = complex(self.coeffs[i].item())
        return PauliTerm(c, PauliString(self.n, x.copy(), z.copy(), k, validate=False))

    def __iter__(self) -> Iterator[PauliTerm]:
        x, z, f, c = self.columns()
        for i in range(len(self)):
            yield PauliTerm(complex(c[i]), PauliString(self.n, x[i].copy(), z[i].copy(),
                                                       int(f[i]), validate=False))

    def labels(self) -> list[str]:
        return [t.string.label for t in self]

    def canonical_key(self, i: int) -> bytes:
        """(z-words, x-words) big-endian key of term i (sums.py:277-280)."""
        t = self.term(i).string
        return t.canonical_key()

    def __eq__(self, other) -> bool:
        if type(other) is not type(self):
            return NotImplemented
        if self.n != other.n or len(self) != len(other):
            return False
        ax, az, af, ac = self.columns()
        bx, bz, bf, bc = other.columns()
        return (np.array_equal(ax, bx) and np.array_equal(az, bz) and np.array_equal(af, bf)
                and np.array_equal(ac, bc))

    __hash__ = None

    def __repr__(self) -> str:
        return f"PauliSumSoA(n={self.n}, terms={len(self)}, device={self.device})"

    def to_aos(self) -> "PauliSum":
        """Inverse of PauliSum.to_soa (sums.py:469-477).  A device sum is
        transposed into packed records on the GPU and comes back in one copy."""
        if self.device.type == "cuda":
            return PauliSum(self.n, _download_aos(self))
        return PauliSum.from_columns(self.n, *self.columns())

    def _check_same_n(self, other) -> None:
        if self.n != other.n:
            raise DimensionError(f"qubit counts differ: {self.n} != {other.n}")

    # ---------------------------------------------------------- operations
    def multiply(self, other, *, threads: int = 1, eps: float = 0.0, combine: bool = True):
        """Outer product; canonical unless combine=False (sums.py:293-305)."""
        self._check_same_n(other)
        other = other if isinstance(other, PauliSumSoA) else other.to_soa()
        return outer_multiply(self, other, eps=eps, combine=combine)

    __mul__ = multiply

    def sort_and_combine(self, eps: float = 0.0):
        """Canonical form: sorted, merged, |c| <= eps dropped (sums.py:286-291)."""
        if eps < 0:
            raise ValueError("eps must be >= 0")
        return sort_combine(self, eps=eps)

    def apply_clifford(self, gate: str, qubits) -> None:
        """Conjugate every term in place; term count unchanged (sums.py:309-316)."""
        from . import gates

        qubits = (int(qubits),) if isinstance(qubits, (int, np.integer)) else tuple(
            int(q) for q in qubits)
        code, q0, q1 = gates.check_gate(gate, qubits, self.n)
        dev, back = _compute_device(self)
        if len(self) == 0:
            return
        S = self.to(dev).planes()
        gates.apply_clifford_planes(S.x, S.z, S.k, S.ld, S.W, S.M, code, q0, q1, dev)
        if back or S.x.data_ptr() != self.x.data_ptr() or S.k.data_ptr() != self.flags.data_ptr():
            self.x.copy_(S.x)
            self.z.copy_(S.z)
            self.flags.copy_(S.k)

    def apply_rotation(self, rot, *, eps: float = 0.0, combine: bool = True):
        """Conjugate by exp(-i*theta/2 * P): at most 2x the terms, canonical
        unless combine=False (sums.py:318-325)."""
        from .rotations import check_rotation_n, rotation_split

        check_rotation_n(self.n, rot)
        dev, back = _compute_device(self)
        with torch.cuda.device(dev):
            if len(self) == 0:
                out = PauliSumSoA.empty(self.n, device=dev)
            else:
                x, z, k, c = rotation_split(self.to(dev).planes(), rot, dev)
                out = _new_sum(self.n, x, z, k, c)
        if combine:
            out = sort_combine(out, eps=eps)
        return _download(out) if back else out

    def truncate(self, eps: float):
        """Drop terms with |coeff| <= eps, keeping order (sums.py:327-339)."""
        if eps < 0:
            raise ValueError("eps must be >= 0")
        keep = torch.abs(self.coeffs) > eps
        out = object.__new__(PauliSumSoA)
        out.n, out.tier = self.n, self.tier
        out.x = self.x[:, keep].contiguous()
        out.z = self.z[:, keep].contiguous()
        out.flags = self.flags[keep].contiguous()
        out.coeffs = self.coeffs[keep].contiguous()
        return out


class PauliSum:
    """Array-of-structures sum on the host, packed records (sums.py:360-426)."""

    __slots__ = ("n", "tier", "_data")

    def __init__(self, n: int, data: np.ndarray | None = None):
        self.n = int(n)
        self.tier = tier_for(self.n)
        dt = aos_dtype(self.tier // 64)
        if data is None:
            data = np.empty(0, dtype=dt)
        if data.dtype != dt:
            raise ValueError(f"expected dtype {dt}, got {data.dtype}")
        _check_finite_np(data["coeff"])
        self._data = data

    @classmethod
    def from_columns(cls, n, x, z, flags, coeffs):
        _check_finite_np(np.asarray(coeffs))
        out = cls(n)
        x = np.asarray(x, dtype=np.uint64)
        data = np.empty(x.shape[0], dtype=aos_dtype(tier_for(n) // 64))
        data["x"], data["z"], data["flags"], data["coeff"] = x, z, flags, coeffs
        out._data = data
        return out

    _from_columns = from_columns

    @classmethod
    def from_terms(cls, entries: Iterable[TermEntry], n: int | None = None):
        return cls.from_columns(*_entries_to_columns(list(entries), n))

    def columns(self):
        d = self._data
        return d["x"], d["z"], d["flags"], d["coeff"]

    _columns = columns

    @property
    def words(self) -> int:
        return self.tier // 64

    def __len__(self) -> int:
        return int(self._data.shape[0])

    @property
    def coeffs(self) -> np.ndarray:
        return self._data["coeff"]

    @property
    def flags(self) -> np.ndarray:
        return self._data["flags"]

    @property
    def x_matrix(self) -> np.ndarray:
        return self._data["x"]

    @property
    def z_matrix(self) -> np.ndarray:
        return self._data["z"]

    @property
    def payload_nbytes(self) -> int:
        return self._data.nbytes

    def term(self, i: int) -> PauliTerm:
        d = self._data[i]
        return PauliTerm(complex(d["coeff"]),
                         PauliString(self.n, d["x"].copy(), d["z"].copy(), int(d["flags"]),
                                     validate=False))

    def __iter__(self):
        return (self.term(i) for i in range(len(self)))

    def labels(self) -> list[str]:
        return [t.string.label for t in self]

    def canonical_key(self, i: int) -> bytes:
        return self.term(i).string.canonical_key()

    def to_soa(self, device=None) -> PauliSumSoA:
        """Transpose into SoA planes (sums.py:417-426).  With a CUDA ``device``
        the packed records are uploaded as they are and transposed on the GPU
        (``pl_aos_to_soa``); without one the result stays on the host."""
        if device is not None and torch.device(device).type == "cuda":
            return _upload_aos(self.n, self._data, torch.device(device))
        d = self._data
        return PauliSumSoA(self.n, np.ascontiguousarray(d["x"].T), np.ascontiguousarray(d["z"].T),
                           d["flags"].copy(), d["coeff"].copy(), device=device, validate=False)

    def __eq__(self, other) -> bool:
        if type(other) is not type(self):
            return NotImplemented
        return self.n == other.n and self._data.tobytes() == other._data.tobytes()

    __hash__ = None

    def __repr__(self) -> str:
        return f"PauliSum(n={self.n}, terms={len(self)})"

    def _check_same_n(self, other) -> None:
        if self.n != other.n:
            raise DimensionError(f"qubit counts differ: {self.n} != {other.n}")

    def multiply(self, other, *, threads: int = 1, eps: float = 0.0, combine: bool = True):
        self._check_same_n(other)
        dev = cuda_device(other.device if isinstance(other, PauliSumSoA) else None)
        b = other.to_soa(dev) if isinstance(other, PauliSum) else other
        return self.to_soa(dev).multiply(b, eps=eps, combine=combine).to_aos()

    __mul__ = multiply

    def sort_and_combine(self, eps: float = 0.0):
        if eps < 0:
            raise ValueError("eps must be >= 0")
        return self.to_soa(cuda_device()).sort_and_combine(eps).to_aos()

    def apply_clifford(self, gate: str, qubits) -> None:
        """In place on the packed records (sums.py:309-316): the records are
        transposed to device planes, conjugated, and written back."""
        soa = self.to_soa()
        soa.apply_clifford(gate, qubits)
        if len(self):
            x, z, f, _ = soa.columns()
            self._data["x"], self._data["z"], self._data["flags"] = x, z, f

    def apply_rotation(self, rot, *, eps: float = 0.0, combine: bool = True):
        """sums.py:318-325."""
        return self.to_soa(cuda_device()).apply_rotation(rot, eps=eps, combine=combine).to_aos()

    def truncate(self, eps: float):
        if eps < 0:
            raise ValueError("eps must be >= 0")
        keep = np.abs(self._data["coeff"]) > eps
        return PauliSum(self.n, self._data[keep].copy())


# ----------------------------------------------------------- kernel drivers
def _compute_device(*sums: PauliSumSoA) -> tuple[torch.device, bool]:
    """The CUDA device to run on and whether results go back to the host."""
    for s in sums:
        if s.device.type == "cuda":
            return s.device, False
    return cuda_device(), True


LAST_PLAN: dict | None = None  # instrumentation: layout of the most recent merge


def _remember(plan) -> None:
    global LAST_PLAN
    LAST_PLAN = {k: int(getattr(plan, k)) for k in
                 ("W", "mode", "n_items", "key_words", "key_bits", "n_buckets", "n_samples",
                  "leaf_cap", "leaf_target", "max_sub", "workspace_bytes")}


LAST_D2H_BYTES = 0  # instrumentation: bytes the most recent _download copied from the device


def _zero_planes(plan) -> tuple[frozenset, frozenset]:
    """Plane words (x, z) that are zero in every term a merge can produce: the
    plan keeps no bit of a canonical-key word whose OR over the operands is
    zero (``seg_len`` 0; key words are z[0..W) then x[0..W), sums.py:104-106),
    and products/merges only XOR and copy operand words."""
    W = int(plan.W)
    zz = frozenset(w for w in range(W) if int(plan.seg_len[w]) == 0)
    zx = frozenset(w for w in range(W) if int(plan.seg_len[W + w]) == 0)
    return zx, zz


def _download(s: PauliSumSoA, zero_x=frozenset(), zero_z=frozenset(),
              zero_flags: bool = False) -> PauliSumSoA:
    """Device result -> host sum through pinned staging buffers (torch's caching
    host allocator recycles them): asynchronous copies, then one sync.

    Planes the caller proves zero (``_zero_planes``; the phase bytes of a
    combined sum) need not cross PCIe: the host clears them while the DMA of
    the other arrays runs, and hands some of them to the DMA engine when it
    runs dry (n=500 sums on 48 qubits: 14 of the 16 planes are zero)."""
    global LAST_D2H_BYTES
    copied = 0

    def pinned_like(t):
        return torch.empty(t.shape, dtype=t.dtype, pin_memory=True)

    def fetch(h, t):
        nonlocal copied
        h.copy_(t, non_blocking=True)
        copied += t.numel() * t.element_size()

    W = s.x.shape[0]
    hx, hz, hk, hc = (pinned_like(t) for t in (s.x, s.z, s.flags, s.coeffs))
    # The DMA engine and the host cores work at the same time, so the
    # proved-zero planes are shared between them dynamically: the host clears
    # plane quarters from the back of the list, and whenever fewer than three
    # copies are outstanding the next one from the front goes to the DMA engine
    # (it is zero on the device too).  Both finish together whatever their
    # rates are at the moment (the host's memory bandwidth is shared).
    m = s.x.shape[1]
    cuts = [0, m] if m < (1 << 22) else [0, m // 4, m // 2, 3 * (m // 4), m]  # finer tail balance
    zeros = [(h[w, a:b], t[w, a:b]) for h, t, zs in ((hx, s.x, zero_x), (hz, s.z, zero_z))
             for w in sorted(zs) for a, b in zip(cuts[:-1], cuts[1:])]
    stream = torch.cuda.current_stream(s.device)

    def mark():
        ev = torch.cuda.Event()
        ev.record(stream)
        return ev

    fetch(hc, s.coeffs)
    for h, t, zero in ((hx, s.x, zero_x), (hz, s.z, zero_z)):
        if not zero:
            fetch(h, t)
        else:
            for w in range(W):
                if w not in zero:
                    fetch(h[w], t[w])
    if not zero_flags:
        fetch(hk, s.flags)
    inflight = [mark()]
    front, back = 0, len(zeros)
    while front < back:
        inflight = [ev for ev in inflight if not ev.query()]
        while len(inflight) < 3 and front < back:
            h, t = zeros[front]
            front += 1
            fetch(h, t)
            inflight.append(mark())
        if front < back:
            back -= 1
            zeros[back][0].zero_()
    if zero_flags:
        hk.zero_()
    torch.cuda.current_stream(s.device).synchronize()
    LAST_D2H_BYTES = copied
    return _new_sum(s.n, hx, hz, hk, hc)


def _upload_aos(n: int, data: np.ndarray, dev: torch.device) -> PauliSumSoA:
    """Packed host records -> device SoA planes: one H2D copy of the records,
    transposed by ``pl_aos_to_soa`` (sums.py:417-426 on the GPU)."""
    W = tier_for(n) // 64
    m = int(data.shape[0])
    if m == 0:
        return PauliSumSoA.empty(n, device=dev)
    raw = np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    if not raw.flags.writeable:
        raw = raw.copy()
    with torch.cuda.device(dev):
        d_raw = torch.from_numpy(raw).to(dev)
        x, z, k, c = _alloc_planes(W, m, dev)
        _native.call("pl_aos_to_soa", W, m, ptr(d_raw), ptr(x), ptr(z), ptr(k), ptr(c),
                     x.stride(0), stream_ptr(dev))
    return _new_sum(n, x, z, k, c)


def _download_aos(s: PauliSumSoA) -> np.ndarray:
    """Device SoA planes -> packed host records (``pl_soa_to_aos`` + one D2H
    copy into pinned memory); the array views that pinned buffer."""
    W, m = s.words, len(s)
    dt = aos_dtype(W)
    if m == 0:
        return np.empty(0, dtype=dt)
    dev = s.device
    S = s.planes()
    with torch.cuda.device(dev):
        rec = torch.empty(m * dt.itemsize, dtype=torch.uint8, device=dev)
        _native.call("pl_soa_to_aos", W, m, ptr(S.x), ptr(S.z), ptr(S.k), ptr(S.c), S.ld,
                     ptr(rec), stream_ptr(dev))
        h = torch.empty(m * dt.itemsize, dtype=torch.uint8, pin_memory=True)
        h.copy_(rec, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
    return h.numpy().view(dt)


def _new_sum(n, x, z, k, c) -> PauliSumSoA:
    out = object.__new__(PauliSumSoA)
    out.n, out.tier = int(n), tier_for(n)
    out.x, out.z, out.flags, out.coeffs = x, z, k, c
    return out


# Merges with more raw items than this run in two phases (merge + count, then
# emit into planes of exactly the merged size): no raw-size output buffers.
# Smaller merges emit into raw-size planes in the same call (no host sync
# between the phases) and are right-sized by _fitted.
_TWO_PHASE_MIN = 1 << 22


def _emit_exact(n, plan, ws, W: int, m: int, dev, st) -> PauliSumSoA:
    x, z, k, c = _alloc_planes(W, m, dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    if m:
        _native.call("pl_merge_emit", C.byref(plan), ptr(ws), ws.numel(), ptr(x), ptr(z), ptr(k),
                     ptr(c), x.stride(0), m, ptr(cnt), st)
    return _new_sum(n, x[:, :m], z[:, :m], k[:m], c[:m])


def _fitted(n, x, z, k, c, m: int) -> PauliSumSoA:
    """The first m merged terms of capacity-sized output planes.  Views are
    kept while they waste at most half the allocation; a heavily merged
    result (e.g. H*H) is copied into right-sized tensors so the raw-size
    buffers are released instead of staying alive with the result."""
    cap = x.shape[1]
    if 2 * m >= cap:
        return _new_sum(n, x[:, :m], z[:, :m], k[:m], c[:m])
    return _new_sum(n, x[:, :m].clone(), z[:, :m].clone(), k[:m].clone(), c[:m].clone())


def _alloc_planes(W: int, cap: int, dev):
    x = torch.empty((W, max(cap, 1)), dtype=torch.int64, device=dev)
    z = torch.empty((W, max(cap, 1)), dtype=torch.int64, device=dev)
    k = torch.empty(max(cap, 1), dtype=torch.uint8, device=dev)
    c = torch.empty(max(cap, 1), dtype=torch.complex128, device=dev)
    return x, z, k, c


def outer_multiply(a: PauliSumSoA, b: PauliSumSoA, *, eps: float = 0.0, combine: bool = True):
    """A*B on the GPU: raw j-major product (sums.py:144-174) or combined
    (sums.py:94-120).  Returns a PauliSumSoA on A's device (host in -> host out).

    Like the reference's multiply, any ``eps`` is accepted: a negative one
    keeps every merged term, exact zeros included (sums.py:113-114)."""
    dev, back = _compute_device(a, b)
    A = a.to(dev).planes()
    B = b.to(dev).planes()
    W, ma, mb = A.W, A.M, B.M
    n_items = ma * mb
    st = stream_ptr(dev)
    zero = ()
    with torch.cuda.device(dev):
        if n_items == 0:
            out = PauliSumSoA.empty(a.n, device=dev)
        elif not combine:
            x, z, k, c = _alloc_planes(W, n_items, dev)
            _native.call("pl_outer_multiply_raw", W, ma, mb,
                         ptr(A.x), ptr(A.z), ptr(A.k), ptr(A.c), A.ld,
                         ptr(B.x), ptr(B.z), ptr(B.k), ptr(B.c), B.ld,
                         ptr(x), ptr(z), ptr(k), ptr(c), x.stride(0), st)
            out = _new_sum(a.n, x, z, k, c)
        else:
            plan = _native.MergePlan()
            _native.call("pl_outer_plan", W, ma, mb, ptr(A.x), ptr(A.z), A.ld, ptr(B.x),
                         ptr(B.z), B.ld, C.byref(plan), st)
            _remember(plan)
            ws = torch.empty(max(int(plan.workspace_bytes), 1), dtype=torch.uint8, device=dev)
            cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            args = (ptr(A.x), ptr(A.z), ptr(A.k), ptr(A.c), A.ld,
                    ptr(B.x), ptr(B.z), ptr(B.k), ptr(B.c), B.ld, float(eps), ptr(ws), ws.numel())
            if n_items > _TWO_PHASE_MIN:
                # merge, read the merged count, then emit into exactly sized planes
                _native.call("pl_outer_multiply_combine", C.byref(plan), *args,
                             None, None, None, None, 0, ptr(cnt), st)
                out = _emit_exact(a.n, plan, ws, W, int(cnt.item()), dev, st)
            else:
                x, z, k, c = _alloc_planes(W, n_items, dev)
                _native.call("pl_outer_multiply_combine", C.byref(plan), *args,
                             ptr(x), ptr(z), ptr(k), ptr(c), x.stride(0), ptr(cnt), st)
                out = _fitted(a.n, x, z, k, c, int(cnt.item()))
            zero = (*_zero_planes(plan), True)  # combined terms carry phase 0
    return _download(out, *zero) if back else out


def sort_combine(s: PauliSumSoA, *, eps: float = 0.0) -> PauliSumSoA:
    """_combine_columns on the GPU (sums.py:94-120).  The public
    sort_and_combine rejects eps < 0 (sums.py:288-289); this internal entry
    (also used by apply_rotation) accepts any eps like _combine_columns."""
    dev, back = _compute_device(s)
    S = s.to(dev).planes()
    W, m = S.W, S.M
    st = stream_ptr(dev)
    zero = ()
    with torch.cuda.device(dev):
        if m == 0:
            out = PauliSumSoA.empty(s.n, device=dev)
        else:
            plan = _native.MergePlan()
            _native.call("pl_sort_plan", W, m, ptr(S.x), ptr(S.z), S.ld, C.byref(plan), st)
            _remember(plan)
            ws = torch.empty(max(int(plan.workspace_bytes), 1), dtype=torch.uint8, device=dev)
            cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            args = (ptr(S.x), ptr(S.z), ptr(S.k), ptr(S.c), S.ld, float(eps), ptr(ws), ws.numel())
            if m > _TWO_PHASE_MIN:
                _native.call("pl_sort_combine", C.byref(plan), *args, None, None, None, None, 0,
                             ptr(cnt), st)
                out = _emit_exact(s.n, plan, ws, W, int(cnt.item()), dev, st)
            else:
                x, z, k, c = _alloc_planes(W, m, dev)
                _native.call("pl_sort_combine", C.byref(plan), *args,
                             ptr(x), ptr(z), ptr(k), ptr(c), x.stride(0), ptr(cnt), st)
                out = _fitted(s.n, x, z, k, c, int(cnt.item()))
            zero = (*_zero_planes(plan), True)
    return _download(out, *zero) if back else out


# ------------------------------------------------------- module functions
def sum_from_terms(entries: Iterable[TermEntry], n: int | None = None) -> PauliSum:
    return PauliSum.from_terms(entries, n)


def sort_and_combine(s, eps: float = 0.0):
    """sums.py:484-485."""
    return s.sort_and_combine(eps)


def sum_multiply(a, b, *, threads: int = 1, eps: float = 0.0, combine: bool = True):
    """sums.py:488-489."""
    return a.multiply(b, threads=threads, eps=eps, combine=combine)


def sum_apply_clifford(s, gate: str, qubits) -> None:
    """sums.py:492-493: conjugate every term of ``s`` in place."""
    s.apply_clifford(gate, qubits)


def sum_apply_rotation(s, rot, *, eps: float = 0.0, combine: bool = True):
    """sums.py:496-497."""
    return s.apply_rotation(rot, eps=eps, combine=combine)


def to_soa(s: PauliSum, device=None) -> PauliSumSoA:
    return s.to_soa(device)


def to_aos(s: PauliSumSoA) -> PauliSum:
    return s.to_aos()


def truncate(s, eps: float):
    return s.truncate(eps)
