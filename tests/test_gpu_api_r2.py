"""GPU: drop-in names added in round 2 against reference-generated fixtures
(tests/golden/make_golden_r2.py): PauliString.apply_clifford /
ps_apply_clifford (strings.py:153-163, :215-216), sum_apply_clifford /
sum_apply_rotation (sums.py:492-497), and a negative eps in multiply /
apply_rotation keeping exact zeros like the reference (sums.py:113-114)."""

import numpy as np
import pytest

import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng
from conftest import golden

pytestmark = pytest.mark.gpu

GATES = [("H", (3,)), ("S", (0,)), ("CNOT", (1, 70)), ("CZ", (65, 2)), ("H", (99,)),
         ("S", 64), ("CNOT", (99, 0)), ("CZ", (10, 11))]


def test_string_apply_clifford_golden(cuda):
    g = golden("string_clifford")
    for t in range(g["x"].shape[0]):
        p = pl.PauliString(100, g["x"][t], g["z"][t], int(g["k"][t]))
        gate, q = GATES[t % len(GATES)]
        o = p.apply_clifford(gate, q) if t % 2 else pl.ps_apply_clifford(p, gate, q)
        assert np.array_equal(o.x, g["ox"][t]) and np.array_equal(o.z, g["oz"][t])
        assert o.phase == int(g["ok"][t])
        assert np.array_equal(p.x, g["x"][t])  # the input string is unchanged


def test_string_apply_clifford_errors(cuda):
    p = pl.PauliString.from_label("XYZ")
    with pytest.raises(IndexError):
        p.apply_clifford("H", 3)
    with pytest.raises(ValueError):
        p.apply_clifford("CNOT", (1, 1))
    with pytest.raises(ValueError):
        p.apply_clifford("T", 0)


def test_sum_apply_wrappers(cuda):
    g = golden("string_clifford")
    s = pl.PauliSumSoA.from_columns(100, g["x"][:8], g["z"][:8], g["k"][:8],
                                    np.ones(8, np.complex128), device=cuda)
    pl.sum_apply_clifford(s, "CNOT", (1, 70))
    exp = [pl.PauliString(100, g["x"][t], g["z"][t], int(g["k"][t])).apply_clifford("CNOT", (1, 70))
           for t in range(8)]
    x, z, k, _ = s.columns()
    assert np.array_equal(x, np.stack([e.x for e in exp]))
    assert np.array_equal(z, np.stack([e.z for e in exp]))
    assert np.array_equal(k, np.array([e.phase for e in exp], np.uint8))
    rot = pl.RotationSpec(pl.PauliString.from_label("X" + "I" * 99), 0.4)
    assert pl.sum_apply_rotation(s, rot) == s.apply_rotation(rot)


def test_negative_eps_keeps_exact_zeros(cuda):
    g = golden("neg_eps")
    H = pl.PauliSumSoA.from_columns(64, g["hx"], g["hz"], g["hf"], g["hc"], device=cuda)
    for out in (pl.sum_multiply(H, H, eps=-1.0), H.multiply(H, eps=-1.0)):
        x, z, k, c = out.columns()
        assert np.array_equal(x, g["ox"]) and np.array_equal(z, g["oz"]) and not k.any()
        assert (c == 0).sum() == (g["oc"] == 0).sum() > 0
        assert np.abs(c - g["oc"]).max() <= 1e-12 * np.abs(g["oc"]).sum()
    rot = pl.RotationSpec(pl.PauliString.from_label(str(g["rot_label"])), np.pi)
    x, z, k, c = H.apply_rotation(rot, eps=-1.0).columns()
    assert np.array_equal(x, g["rx"]) and np.array_equal(z, g["rz"]) and not k.any()
    assert np.abs(c - g["rc"]).max() <= 1e-12 * np.abs(g["rc"]).sum()
    with pytest.raises(ValueError):
        pl.sort_and_combine(H, eps=-1.0)  # the public sort_and_combine still rejects it


@pytest.mark.parametrize("n", [40, 100, 200, 500, 1000])
@pytest.mark.parametrize("m", [0, 1, 15, 128, 129, 1000])
def test_aos_soa_device_transpose(cuda, n, m):
    """f4: packed records <-> device planes (sums.py:417-426, :469-477) is the
    exact bijection the host transposes compute, at every tier and across
    tile boundaries (tiles of 128 records)."""
    x, z, f, c = rng.random_columns(n, max(m, 1), 11)
    x, z, f, c = x[:m], z[:m], f[:m], c[:m]
    f = (np.arange(m) % 4).astype(np.uint8)
    aos = pl.PauliSum.from_columns(n, x, z, f, c)
    dev_soa = aos.to_soa(device=cuda)
    assert dev_soa.device.type == "cuda" and len(dev_soa) == m
    host_soa = aos.to_soa()
    assert dev_soa.cpu() == host_soa
    back = dev_soa.to_aos()
    assert isinstance(back, pl.PauliSum) and back == aos


def test_aos_multiply_runs_on_device_records(cuda):
    """PauliSum.multiply uploads the records, multiplies on the GPU and returns
    records transposed on the GPU: same terms as the SoA path."""
    a, b = rng.config_columns(2, scale=0.2)
    A, B = pl.PauliSum.from_columns(500, *a), pl.PauliSum.from_columns(500, *b)
    got = A.multiply(B)
    ref = pl.sum_multiply(pl.PauliSumSoA.from_columns(500, *a, device=cuda),
                          pl.PauliSumSoA.from_columns(500, *b, device=cuda))
    assert got == ref.cpu().to_aos()
    assert A.sort_and_combine() == pl.sort_and_combine(
        pl.PauliSumSoA.from_columns(500, *a, device=cuda)).cpu().to_aos()
