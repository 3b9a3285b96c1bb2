"""§8(f) rows f1/f2 on the CPU: the oracle restatement pinned to fixtures made
by running the reference (tests/golden/make_golden_f12.py), and the host-side
logic of the drop-in (trig snapping, RotationSpec, gate validation)."""

import math

import numpy as np
import pytest

from conftest import golden
from oracle import numpy_ref as R
from paper_2605_25974_b200 import gates, rotations

CLIFF = ["clifford_n40", "clifford_n100", "clifford_n500", "clifford_n1000"]
ROTS = [("rotation_n100", 100), ("rotation_n500", 500), ("rotation_n5", 5)]


@pytest.mark.parametrize("name", CLIFF)
def test_oracle_clifford_golden(name):
    g = golden(name)
    n = {"clifford_n40": 40, "clifford_n100": 100, "clifford_n500": 500, "clifford_n1000": 1000}[name]
    x, z, f = g["x0"], g["z0"], g["f0"]
    for s in range(len(g["gates"])):
        gate = str(g["gates"][s])
        q = (int(g["q0"][s]),) if g["q1"][s] < 0 else (int(g["q0"][s]), int(g["q1"][s]))
        x, z, f = R.apply_clifford(x, z, f, gate, q, n)
        assert np.array_equal(x, g["xs"][s]) and np.array_equal(z, g["zs"][s])
        assert np.array_equal(f, g["fs"][s])


@pytest.mark.parametrize("name,n", ROTS)
def test_oracle_rotation_golden(name, n):
    g = golden(name)
    for t, theta in enumerate(g["theta"]):
        cos_t, sin_t = rotations.trig_values(float(theta))
        assert (cos_t, sin_t) == tuple(g[f"trig{t}"])
        ox, oz, of, oc = R.rotation_split(g["x0"], g["z0"], g["f0"], g["c0"], g["gx"][t],
                                          g["gz"][t], cos_t, sin_t)
        assert np.array_equal(ox, g[f"sx{t}"]) and np.array_equal(oz, g[f"sz{t}"])
        assert np.array_equal(of, g[f"sf{t}"])
        np.testing.assert_allclose(oc, g[f"sc{t}"], rtol=1e-15, atol=0)
        cx, cz, cf, cc = R.combine(ox, oz, of, oc)
        assert np.array_equal(cx, g[f"cx{t}"]) and np.array_equal(cz, g[f"cz{t}"])
        scale = max(float(np.abs(g[f"cc{t}"]).sum()), 1e-300)
        assert float(np.abs(cc - g[f"cc{t}"]).max(initial=0)) <= 1e-12 * scale


def test_rotation_n5_merges():
    g = golden("rotation_n5")
    assert len(g["cx0"]) < len(g["sx0"])  # products collide with existing strings


def test_trig_snap():
    assert rotations.trig_values(math.pi) == (-1.0, 0.0)
    assert rotations.trig_values(math.pi / 2) == (0.0, 1.0)
    assert rotations.trig_values(0.0) == (1.0, 0.0)
    c, s = rotations.trig_values(0.3)
    assert c == math.cos(0.3) and s == math.sin(0.3)


def test_rotation_spec_phases():
    from paper_2605_25974_b200.strings import PauliString

    p = PauliString.from_label("XZY", phase=2)
    r = rotations.RotationSpec(p, 0.7)
    assert r.generator.phase == 0 and r.theta == -0.7
    with pytest.raises(ValueError):
        rotations.RotationSpec(PauliString.from_label("XZY", phase=1), 0.7)


def test_gate_validation():
    assert gates.check_gate("h", (3,), 10) == (0, 3, -1)
    assert gates.check_gate("CNOT", (1, 9), 10) == (2, 1, 9)
    with pytest.raises(IndexError):
        gates.check_gate("S", (10,), 10)
    with pytest.raises(ValueError):
        gates.check_gate("CZ", (2, 2), 10)
    with pytest.raises(ValueError):
        gates.check_gate("H", (1, 2), 10)
    with pytest.raises(ValueError):
        gates.check_gate("T", (1,), 10)


# ------------------------------------------------------------------ f4 hamio
def test_hamio_write_matches_reference():
    import io

    import paper_2605_25974_b200 as pl

    g = golden("hamio_n12")
    s = pl.PauliSum.from_columns(12, g["x0"], g["z0"], g["f0"], g["c0"])
    buf = io.StringIO()
    pl.write_hamiltonian(buf, s)
    assert buf.getvalue() == str(g["text"])


def test_hamio_read_matches_reference():
    import io

    import paper_2605_25974_b200 as pl

    g = golden("hamio_n12")
    s = pl.read_hamiltonian(io.StringIO(str(g["src"])))
    x, z, f, c = s.columns()
    assert np.array_equal(x, g["px"]) and np.array_equal(z, g["pz"])
    assert np.array_equal(f, g["pf"]) and np.array_equal(c, g["pc"])


@pytest.mark.parametrize("text,exc", [
    ("1.0 0.0\n", "HamiltonianFormatError"),
    ("1.0 abc XY\n", "HamiltonianFormatError"),
    ("1.0 0.0 XY\n2.0 0.0 XYZ\n", "DimensionError"),
    ("1.0 0.0 XQ\n", "HamiltonianFormatError"),
    ("# nothing\n\n", "HamiltonianFormatError"),
])
def test_hamio_errors(text, exc):
    import io

    import paper_2605_25974_b200 as pl

    with pytest.raises(getattr(pl, exc)) as e:
        pl.read_hamiltonian(io.StringIO(text))
    if exc == "HamiltonianFormatError":
        assert e.value.line in (0, 1, 2)


# ------------------------------------------------------------ f3 parallel grouping
@pytest.mark.parametrize("name", ["group_par_rand", "group_par_dense", "group_par_jw"])
@pytest.mark.parametrize("chunks", [1, 2, 5, 16])
def test_oracle_greedy_parallel_golden(name, chunks):
    g = golden(name)
    groups, checks = R.greedy_parallel(g["x"], g["z"], chunks)
    flat = [t for grp in groups for t in grp]
    offs = np.cumsum([0] + [len(grp) for grp in groups])
    assert np.array_equal(flat, g[f"members{chunks}"])
    assert np.array_equal(offs, g[f"offsets{chunks}"])
    assert checks == int(g[f"checks{chunks}"])
