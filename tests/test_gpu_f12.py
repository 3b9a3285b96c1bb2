"""GPU parity for the §8(f) rows f1 (rotation split + combine) and f2
(Clifford conjugation): bit-exact letters / phases / split coefficients
against fixtures made by the reference, combined coefficients within 1e-12
of the summed magnitudes; size-independent properties at 10^6 terms."""

import math

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import numpy_ref as R
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng
from paper_2605_25974_b200.strings import PauliString

pytestmark = pytest.mark.gpu

CLIFF = [("clifford_n40", 40), ("clifford_n100", 100), ("clifford_n500", 500),
         ("clifford_n1000", 1000)]
ROTS = [("rotation_n100", 100), ("rotation_n500", 500), ("rotation_n5", 5)]


def steps(g):
    for s in range(len(g["gates"])):
        gate = str(g["gates"][s])
        q = (int(g["q0"][s]),) if g["q1"][s] < 0 else (int(g["q0"][s]), int(g["q1"][s]))
        yield s, gate, q


@pytest.mark.parametrize("name,n", CLIFF)
def test_clifford_golden_soa(cuda, name, n):
    g = golden(name)
    s = pl.PauliSumSoA.from_columns(n, g["x0"], g["z0"], g["f0"], g["c0"], device=cuda)
    for t, gate, q in steps(g):
        s.apply_clifford(gate, q if len(q) > 1 else q[0])
        x, z, f, c = s.columns()
        assert np.array_equal(x, g["xs"][t]) and np.array_equal(z, g["zs"][t]), (t, gate, q)
        assert np.array_equal(f, g["fs"][t]), (t, gate, q)
        assert np.array_equal(c, g["c0"])


def test_clifford_golden_aos_host(cuda):
    g = golden("clifford_n500")
    s = pl.PauliSum.from_columns(500, g["x0"], g["z0"], g["f0"], g["c0"])
    for t, gate, q in steps(g):
        s.apply_clifford(gate, q)
    x, z, f, _ = s.columns()
    assert np.array_equal(x, g["xs"][-1]) and np.array_equal(z, g["zs"][-1])
    assert np.array_equal(f, g["fs"][-1])


def test_clifford_errors(cuda):
    s = pl.PauliSumSoA.from_columns(10, *rng.random_columns(10, 4, 1), device=cuda)
    with pytest.raises(IndexError):
        s.apply_clifford("H", 10)
    with pytest.raises(ValueError):
        s.apply_clifford("CNOT", (3, 3))


def test_clifford_involutions_large(cuda):
    """H^2 = S^4 = CNOT^2 = CZ^2 = identity on 10^6 terms (phases included)."""
    x, z, f, c = rng.random_columns(500, 1 << 20, 5)
    f = np.random.default_rng(1).integers(0, 4, len(f)).astype(np.uint8)
    s = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=cuda)
    for gate, q, reps in (("H", 77, 2), ("S", 300, 4), ("CNOT", (3, 64), 2), ("CZ", (5, 6), 2),
                          ("CNOT", (499, 0), 2)):
        for _ in range(reps):
            s.apply_clifford(gate, q)
    ox, oz, of, _ = s.columns()
    assert np.array_equal(ox, x) and np.array_equal(oz, z) and np.array_equal(of, f)


def test_clifford_matches_oracle_large(cuda):
    x, z, f, c = rng.random_columns(100, 200_000, 9)
    f = np.random.default_rng(2).integers(0, 4, len(f)).astype(np.uint8)
    s = pl.PauliSumSoA.from_columns(100, x, z, f, c, device=cuda)
    for gate, q in (("H", (70,)), ("S", (3,)), ("CNOT", (10, 90)), ("CZ", (64, 65))):
        s.apply_clifford(gate, q)
        x, z, f = R.apply_clifford(x, z, f, gate, q, 100)
    ox, oz, of, _ = s.columns()
    assert np.array_equal(ox, x) and np.array_equal(oz, z) and np.array_equal(of, f)


@pytest.mark.parametrize("name,n", ROTS)
def test_rotation_golden(cuda, name, n):
    g = golden(name)
    s = pl.PauliSumSoA.from_columns(n, g["x0"], g["z0"], g["f0"], g["c0"], device=cuda)
    for t, theta in enumerate(g["theta"]):
        rot = pl.RotationSpec(PauliString(n, g["gx"][t], g["gz"][t], 0), float(theta))
        raw = s.apply_rotation(rot, combine=False)
        x, z, f, c = raw.columns()
        assert np.array_equal(x, g[f"sx{t}"]) and np.array_equal(z, g[f"sz{t}"]), t
        assert np.array_equal(f, g[f"sf{t}"]), t
        assert np.array_equal(c, g[f"sc{t}"]), t  # numpy complex products, bit for bit
        comb = s.apply_rotation(rot)
        x, z, f, c = comb.columns()
        assert np.array_equal(x, g[f"cx{t}"]) and np.array_equal(z, g[f"cz{t}"]), t
        assert not f.any()
        scale = max(float(np.abs(g[f"cc{t}"]).sum()), 1e-300)
        assert float(np.abs(c - g[f"cc{t}"]).max(initial=0)) <= 1e-12 * scale, t


def test_rotation_host_in_host_out(cuda):
    g = golden("rotation_n100")
    s = pl.PauliSum.from_columns(100, g["x0"], g["z0"], g["f0"], g["c0"])
    rot = pl.RotationSpec(PauliString(100, g["gx"][0], g["gz"][0], 0), float(g["theta"][0]))
    out = s.apply_rotation(rot)
    x, z, _, _ = out.columns()
    assert np.array_equal(x, g["cx0"]) and np.array_equal(z, g["cz0"])


def test_rotation_large_counts(cuda):
    """Split size = M + #anti-commuting terms (batch_sip), 2^20 terms."""
    x, z, f, c = rng.random_columns(500, 1 << 20, 12)
    s = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=cuda)
    gx, gz, _, _ = rng.random_columns(500, 1, 99)
    rot = pl.RotationSpec(PauliString(500, gx[0], gz[0], 0), 0.4)
    anti = int(R.sip(x, z, np.broadcast_to(gx[0], x.shape), np.broadcast_to(gz[0], z.shape)).sum())
    raw = s.apply_rotation(rot, combine=False)
    assert len(raw) == len(x) + anti
    exp = R.rotation_split(x[:4096], z[:4096], f[:4096], c[:4096], gx[0], gz[0],
                           *pl.trig_values(0.4))
    sub = pl.PauliSumSoA.from_columns(500, x[:4096], z[:4096], f[:4096], c[:4096], device=cuda)
    got = sub.apply_rotation(rot, combine=False).columns()
    for a, b in zip(got, exp):
        assert np.array_equal(a, b)


def test_rotation_dimension_error(cuda):
    s = pl.PauliSumSoA.from_columns(10, *rng.random_columns(10, 4, 1), device=cuda)
    rot = pl.RotationSpec(PauliString.from_label("XYZ"), 0.1)
    with pytest.raises(pl.DimensionError):
        s.apply_rotation(rot)


def test_reorder_rotation_known_answer(cuda):
    # X past a quarter turn about Z: anticommute -> i*Z*X = i*(iY) = -Y -> theta flips sign
    r = pl.RotationSpec(PauliString.from_label("X"), 0.3)
    out = pl.reorder_rotation(r, PauliString.from_label("Z"))
    assert out.generator.label == "Y" and out.theta == -0.3
    same = pl.reorder_rotation(r, PauliString.from_label("X"))
    assert same is r
