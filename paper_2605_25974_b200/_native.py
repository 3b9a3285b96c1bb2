"""ctypes binding of ``libpaulib_b200.so`` (the C ABI in include/paulib_b200.h).

This is the only route from the Python layer to the hot path: there is no
CPU fallback.  If the library is missing or fails to load, every device
operation raises :class:`NativeLibraryError`.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libpaulib_b200.so"

PL_PLAN_MAX_SEG = 32


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing or returned an error."""


class MergePlan(C.Structure):
    """Mirror of ``pl_merge_plan``."""

    _fields_ = [
        ("W", C.c_int32),
        ("mode", C.c_int32),
        ("ma", C.c_int64),
        ("mb", C.c_int64),
        ("n_items", C.c_int64),
        ("key_words", C.c_int32),
        ("key_bits", C.c_int32),
        ("seg_lo", C.c_int32 * PL_PLAN_MAX_SEG),
        ("seg_len", C.c_int32 * PL_PLAN_MAX_SEG),
        ("seg_pos", C.c_int32 * PL_PLAN_MAX_SEG),
        ("n_buckets", C.c_int32),
        ("n_samples", C.c_int32),
        ("leaf_cap", C.c_int32),
        ("leaf_target", C.c_int32),
        ("max_sub", C.c_int32),
        ("pad0", C.c_int32),
        ("workspace_bytes", C.c_int64),
        ("reserved", C.c_int64 * 8),
    ]


_P = C.c_void_p
_I = C.c_int
_L = C.c_int64
_D = C.c_double
_S = C.c_size_t

# name -> (restype, argtypes); the exported surface of include/paulib_b200.h
SIGNATURES = {
    "pl_last_error": (C.c_char_p, []),
    "pl_abi_version": (_I, []),
    "pl_batch_multiply": (_I, [_I, _L, _P, _P, _P, _L, _P, _P, _P, _L, _P, _P, _P, _L, _P]),
    "pl_batch_sip": (_I, [_I, _L, _P, _P, _L, _P, _P, _L, _P, _P]),
    "pl_pair_host": (_I, [_I, _P, _P, _I, _P, _P, _I, _P, _P, _P, _P, _P]),
    "pl_outer_multiply_raw": (_I, [_I, _L, _L, _P, _P, _P, _P, _L, _P, _P, _P, _P, _L,
                                   _P, _P, _P, _P, _L, _P]),
    "pl_outer_plan": (_I, [_I, _L, _L, _P, _P, _L, _P, _P, _L, C.POINTER(MergePlan), _P]),
    "pl_sort_plan": (_I, [_I, _L, _P, _P, _L, C.POINTER(MergePlan), _P]),
    "pl_outer_multiply_combine": (_I, [C.POINTER(MergePlan), _P, _P, _P, _P, _L, _P, _P, _P, _P,
                                       _L, _D, _P, _S, _P, _P, _P, _P, _L, _P, _P]),
    "pl_sort_combine": (_I, [C.POINTER(MergePlan), _P, _P, _P, _P, _L, _D, _P, _S, _P, _P, _P,
                             _P, _L, _P, _P]),
    "pl_commutation_bitmatrix": (_I, [_I, _L, _P, _P, _L, _L, _L, _L, _L, _P, _L, _I, _P, _S,
                                      _P]),
    "pl_bitmatrix_workspace_bytes": (_L, [_I, _L]),
    "pl_group_workspace_bytes": (_L, [_I, _L]),
    "pl_group_greedy": (_I, [_I, _L, _P, _P, _L, _P, _P, _P, _P, _S, _P]),
    "pl_aos_to_soa": (_I, [_I, _L, _P, _P, _P, _P, _P, _L, _P]),
    "pl_soa_to_aos": (_I, [_I, _L, _P, _P, _P, _P, _L, _P, _P]),
    "pl_merge_emit": (_I, [C.POINTER(MergePlan), _P, _S, _P, _P, _P, _P, _L, _L, _P, _P]),
    "pl_dist_item_bytes": (_I, [C.POINTER(MergePlan)]),
    "pl_dist_workspace_bytes": (_L, [C.POINTER(MergePlan), _L, C.c_int32]),
    "pl_outer_partition": (_I, [C.POINTER(MergePlan), _P, _P, _P, _L, _P, _P, _P, _L, _L, _L,
                                _P, _S, _P, _P, _P]),
    "pl_merge_received": (_I, [C.POINTER(MergePlan), _P, _L, _P, _I, C.c_int32, C.c_int32,
                               _P, _P, _P, _P, _L, _P, _P, _P, _P, _L, _D, _P, _S,
                               _P, _P, _P, _P, _L, _P, _P]),
    "pl_group_merge_workspace_bytes": (_L, [_L, C.c_int32]),
    "pl_group_merge": (_I, [_I, _L, _P, _P, _L, _P, _P, C.c_int32, _P, _P, _P, _P, _S, _P]),
    "pl_apply_clifford": (_I, [_I, _L, _P, _P, _P, _L, _I, _I, _I, _P]),
    "pl_rotation_workspace_bytes": (_L, [_L]),
    "pl_rotation_split": (_I, [_I, _L, _P, _P, _P, _P, _L, _P, _P, _D, _D, _D, _P, _S, _P, _P, _P,
                               _P, _L, _P, _P]),
    "pl_stage_timing": (_I, [_I]),
    "pl_stage_times": (_I, [_P, _P, _I]),
}


def stage_timing(enable: bool) -> None:
    load().pl_stage_timing(1 if enable else 0)


def stage_times(max_stages: int = 4096) -> list[tuple[str, float]]:
    """(kernel name, ms) for every kernel launched since timing was enabled."""
    names = C.create_string_buffer(32 * max_stages)
    ms = (C.c_float * max_stages)()
    n = load().pl_stage_times(names, ms, max_stages)
    raw = names.raw
    return [(raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(), float(ms[i])) for i in range(n)]

_lib = None
_load_error: str | None = None


def library_path() -> Path:
    return _LIB_PATH


def load(required: bool = True):
    """Load (once) and return the ctypes library handle."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is None:
        if not _LIB_PATH.exists():
            _load_error = (f"{_LIB_PATH.name} not built; run __graft_entry__.build() or "
                           f"python -m paper_2605_25974_b200._build")
        else:
            try:
                lib = C.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
                return _lib
            except OSError as e:  # pragma: no cover - depends on the box
                _load_error = f"cannot load {_LIB_PATH}: {e}"
            except AttributeError as e:
                _load_error = f"{_LIB_PATH.name} lacks a symbol: {e}"
    if required:
        raise NativeLibraryError(_load_error)
    return None


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().pl_last_error().decode(errors="replace")
        raise NativeLibraryError(f"{what} failed (code {rc}): {msg}")


def call(name: str, *args):
    """Call an exported function and raise on a nonzero status."""
    rc = getattr(load(), name)(*args)
    check(rc, name)
    return rc
