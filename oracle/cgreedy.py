"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/greedy.c (grouping.py:67-83)."""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "libgreedy_oracle.so"
_lib = None


def build() -> Path:
    if not _SO.exists() or _SO.stat().st_mtime < (_HERE / "greedy.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(str(_SO))
        lib.oracle_greedy.restype = C.c_int64
        lib.oracle_greedy.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]
        _lib = lib
    return _lib


def greedy(x: np.ndarray, z: np.ndarray):
    """(group_of int32 (M,), n_groups, pair_checks) for term-major (M, W) words."""
    x = np.ascontiguousarray(x, dtype=np.uint64)
    z = np.ascontiguousarray(z, dtype=np.uint64)
    m, W = x.shape
    gof = np.zeros(m, dtype=np.int32)
    pc = np.zeros(1, dtype=np.int64)
    ng = _load().oracle_greedy(W, m, x.ctypes.data, z.ctypes.data, gof.ctypes.data, pc.ctypes.data)
    if ng < 0:
        raise MemoryError("oracle_greedy allocation failed")
    return gof, int(ng), int(pc[0])
