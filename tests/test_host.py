"""CPU: host-side logic (tiers, labels, generators) and the C-ABI library surface."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import bits, rng
from paper_2605_25974_b200 import _native
from paper_2605_25974_b200.strings import PauliString
from paper_2605_25974_b200.sums import PauliSum, PauliSumSoA


def test_tiers():
    assert bits.tier_for(1) == 64 and bits.tier_for(64) == 64 and bits.tier_for(65) == 128
    assert bits.words_for(500) == 8 and bits.words_for(100) == 2 and bits.words_for(1024) == 16
    with pytest.raises(bits.CapacityError):
        bits.tier_for(1025)
    with pytest.raises(ValueError):
        bits.tier_for(0)


def test_labels_roundtrip_and_errors():
    p = PauliString.from_label("XIZY", 2)
    assert p.to_label() == ("XIZY", 2)
    assert int(p.x[0]) == 0b1001 and int(p.z[0]) == 0b1100
    assert PauliString.from_label("XIZ").x[0] == 1 and PauliString.from_label("XIZ").z[0] == 4
    with pytest.raises(bits.LabelError):
        PauliString.from_label("XAZ")
    with pytest.raises(bits.LabelError):
        PauliString.from_label("")
    with pytest.raises(bits.CapacityError):
        PauliString.from_label("I" * 1025)
    long = "XYZI" * 125
    assert PauliString.from_label(long).label == long
    assert PauliString.from_label("XZ").canonical_key() == (
        np.array([2], ">u8").tobytes() + np.array([1], ">u8").tobytes())


def test_padding_check():
    with pytest.raises(ValueError):
        PauliString(3, np.array([8], np.uint64), np.array([0], np.uint64))


@pytest.mark.parametrize("n,seed", [(500, 0), (100, 7)])
def test_random_columns_match_reference(n, seed):
    g = golden(f"rng_n{n}_s{seed}")
    x, z, f, c = rng.random_columns(n, g["x"].shape[0], seed)
    assert np.array_equal(x, g["x"]) and np.array_equal(z, g["z"])
    assert np.array_equal(f, g["f"]) and np.array_equal(c, g["c"])


def test_splitmix_stream_continuity():
    a = rng.SplitMix64(42)
    first = a.next_array(5)
    second = a.next_array(3)
    b = rng.SplitMix64(42).next_array(8)
    assert np.array_equal(np.concatenate([first, second]), b)


def test_config_generators_shapes():
    (a, b) = rng.config_columns(2, scale=0.05)
    assert a[0].shape == (50, 8)
    w = np.bitwise_count(a[0] | a[1]).sum(axis=1)
    assert (w == 4).all()
    assert not (a[0][:, 1:] | a[1][:, 1:]).any()           # support inside qubits 0..23
    assert not ((a[0][:, 0] | a[1][:, 0]) >> np.uint64(24)).any()
    (c, d) = rng.config_columns(4, scale=0.01)
    assert (np.bitwise_count(c[0] | c[1]).sum(axis=1) == 8).all()
    x, z, _, coef = rng.config_columns(3, scale=0.01)
    assert x.shape == (1000, 2) and np.isreal(coef).all()
    x5, z5, _, c5 = rng.c5_columns(2000, seed=4)
    wt = np.bitwise_count(x5 | z5).sum(axis=1)
    assert wt.min() >= 2 and wt.max() <= 12
    # 10% exact duplicates (string and coefficient)
    keys = np.concatenate([x5, z5, c5.view(np.uint64).reshape(-1, 2)], axis=1)
    assert len(np.unique(keys, axis=0)) <= 1800 + 10


def test_jw_structure():
    x, z, _, _ = rng.jw_columns(100, 500, 2)
    bits_x = bits.words_to_bits(x, 100)
    bits_z = bits.words_to_bits(z, 100)
    for t in range(500):
        xs = np.flatnonzero(bits_x[t])
        if xs.size == 0:
            assert 1 <= bits_z[t].sum() <= 2
        else:
            assert xs.size in (2, 4)
            for p in range(0, xs.size, 2):
                lo, hi = xs[p], xs[p + 1]
                assert bits_z[t, lo + 1:hi].all()


def test_sum_layouts_host():
    s = PauliSum.from_terms([(1.0, "XIZ"), (0.5j, "YYI")])
    soa = s.to_soa()
    assert soa.x.shape == (1, 2) and soa.device.type == "cpu"
    assert soa.to_aos() == s
    assert s.labels() == ["XIZ", "YYI"]
    with pytest.raises(ValueError):
        PauliSum.from_terms([(float("nan"), "X")])
    with pytest.raises(bits.DimensionError):
        PauliSum.from_terms([(1, "X"), (1, "XX")])


HEADER = ROOT / "include" / "paulib_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(pl_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    lib_path = _native.library_path()
    if not lib_path.exists():
        from paper_2605_25974_b200._build import build_native

        build_native()
    lib = ctypes.CDLL(str(lib_path))
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in paulib_b200.h but not exported"
    assert set(syms) <= set(_native.SIGNATURES), "ctypes binding misses a declared symbol"
    assert _native.load().pl_abi_version() == 1


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    s = PauliSumSoA.from_terms([(1.0, "XZ")])
    with pytest.raises(_native.NativeLibraryError):
        s.multiply(s)


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2605_25974_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", f.read_text(), re.M), f


def test_random_string_matches_reference():
    """rng.random_string (rng.py:66-70) against reference-generated strings."""
    g = golden("rng_string")
    for n, seed in ((5, 0), (100, 7), (500, 3)):
        st = pl.SplitMix64(seed)
        for t in range(3):
            p = pl.random_string(n, st)
            assert p.n == n and p.phase == 0
            assert np.array_equal(p.x, g[f"x_{n}_{seed}"][t])
            assert np.array_equal(p.z, g[f"z_{n}_{seed}"][t])
        assert st.next_uint64() == int(g[f"next_{n}_{seed}"])


REFERENCE_ALL = [  # paulialg/__init__.py:52-96
    "CAPACITY_TIERS", "MAX_QUBITS", "CapacityError", "CommutationPartition", "DimensionError",
    "GroupingStats", "HamiltonianFormatError", "LabelError", "PauliString", "PauliSum",
    "PauliSumSoA", "PauliTerm", "RotationSpec", "SplitMix64", "ValidationReport",
    "group_greedy", "group_greedy_parallel", "product_phase_exponent", "ps_apply_clifford",
    "ps_commutes", "ps_from_label", "ps_multiply", "ps_to_label", "ps_weight", "random_string",
    "random_sum", "read_hamiltonian", "reorder_rotation", "sort_and_combine",
    "sum_apply_clifford", "sum_apply_rotation", "sum_from_terms", "sum_multiply",
    "symplectic_inner_product", "tier_for", "to_aos", "to_soa", "truncate",
    "validate_partition", "write_hamiltonian", "__version__"]


def test_reference_exports_present():
    missing = [nm for nm in REFERENCE_ALL if not hasattr(pl, nm) or nm not in pl.__all__]
    assert not missing, missing
    assert isinstance(pl.random_sum(6, 3, 1), pl.PauliSum)  # the reference returns AoS


def test_hamio_bulk_roundtrip_host():
    import io

    x, z, _, c = pl.random_columns(70, 300, 5)
    f = (np.arange(300) % 4).astype(np.uint8)
    s = pl.PauliSum.from_columns(70, x, z, f, c * (1 + 0.5j))
    buf = io.StringIO()
    pl.write_hamiltonian(buf, s)
    back = pl.read_hamiltonian(io.StringIO(buf.getvalue()))
    bx, bz, bf, bc = back.columns()
    assert np.array_equal(bx, x) and np.array_equal(bz, z) and not bf.any()
    assert np.array_equal(bc, np.asarray(c * (1 + 0.5j)) * pl.PHASE_FACTORS[f])
