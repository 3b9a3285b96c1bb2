"""Clifford conjugation in place (§8(f) row f2), the reference's
``paulialg/gates.py`` (apply_clifford_inplace, gates.py:72-102) on device SoA
planes: only the plane words holding the touched qubits are streamed."""

from __future__ import annotations

from typing import Sequence

from . import _native
from ._device import ptr, stream_ptr

GATES_1Q = ("H", "S")
GATES_2Q = ("CNOT", "CZ")
_CODE = {"H": 0, "S": 1, "CNOT": 2, "CZ": 3}


def _locate(q: int, n: int) -> tuple[int, int]:
    """gates.py:21-24."""
    if not 0 <= q < n:
        raise IndexError(f"qubit index {q} out of range for {n} qubits")
    return q // 64, q % 64


def check_gate(gate: str, qubits: Sequence[int], n: int) -> tuple[int, int, int]:
    """Validation of apply_clifford_inplace (gates.py:82-102): returns
    (gate code, q0, q1) or raises the reference's exceptions."""
    gate = gate.upper()
    if gate in GATES_1Q:
        if len(qubits) != 1:
            raise ValueError(f"{gate} takes one qubit index, got {len(qubits)}")
        _locate(qubits[0], n)
        return _CODE[gate], int(qubits[0]), -1
    if gate in GATES_2Q:
        if len(qubits) != 2:
            raise ValueError(f"{gate} takes two qubit indices, got {len(qubits)}")
        c, t = qubits
        if c == t:
            raise ValueError(f"{gate} requires distinct qubits, got ({c}, {t})")
        _locate(c, n)
        _locate(t, n)
        return _CODE[gate], int(c), int(t)
    raise ValueError(f"unknown Clifford gate {gate!r}; expected one of H, S, CNOT, CZ")


def apply_clifford_planes(x, z, k, ld: int, W: int, m: int, code: int, q0: int, q1: int, dev):
    """pl_apply_clifford on device planes (in place)."""
    _native.call("pl_apply_clifford", W, m, ptr(x), ptr(z), ptr(k), ld, code, q0, q1,
                 stream_ptr(dev))
