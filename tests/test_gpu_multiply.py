"""GPU parity: K1 batched multiply, single-string algebra, raw outer product."""

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import numpy_ref as R
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng
from paper_2605_25974_b200._device import i64_tensor_to_u64, u64_to_i64_tensor

pytestmark = pytest.mark.gpu


def planes(a, dev):
    return u64_to_i64_tensor(np.ascontiguousarray(a.T)).to(dev)


def host_cols(t):
    return np.ascontiguousarray(i64_tensor_to_u64(t).T)


@pytest.mark.parametrize("n", [40, 100, 200, 500, 1000])
def test_batch_multiply_golden(cuda, n):
    g = golden(f"batch_n{n}")
    ox, oz, ok = pl.batch_multiply(planes(g["ax"], cuda), planes(g["az"], cuda),
                                   torch.from_numpy(g["af"]).to(cuda), planes(g["bx"], cuda),
                                   planes(g["bz"], cuda), torch.from_numpy(g["bf"]).to(cuda))
    assert np.array_equal(host_cols(ox), g["ox"]) and np.array_equal(host_cols(oz), g["oz"])
    assert np.array_equal(ok.cpu().numpy(), g["ok"])


@pytest.mark.parametrize("P", [1, 2, 3, 31, 65536, 65537])
def test_batch_multiply_config1_and_odd(cuda, P):
    ax, az, _, _ = rng.random_columns(500, P, 0)
    bx, bz, _, _ = rng.random_columns(500, P, 1)
    r = np.random.default_rng(P)
    af = r.integers(0, 4, P).astype(np.uint8)
    bf = r.integers(0, 4, P).astype(np.uint8)
    ex, ez, ek = R.batch_pair_multiply(ax, az, af, bx, bz, bf)
    x, z, k = pl.batch_pair_multiply(ax, az, af, bx, bz, bf)      # host drop-in path
    assert np.array_equal(x, ex) and np.array_equal(z, ez) and np.array_equal(k, ek)


def test_batch_multiply_unaligned_views(cuda):
    """Odd offsets force the scalar (non-128-bit) path."""
    P = 1001
    ax, az, _, _ = rng.random_columns(500, P + 1, 3)
    bx, bz, _, _ = rng.random_columns(500, P + 1, 4)
    A = [planes(v, cuda)[:, 1:] for v in (ax, az)]
    B = [planes(v, cuda)[:, 1:] for v in (bx, bz)]
    x, z, k = pl.batch_multiply(A[0], A[1], None, B[0], B[1], None)
    ex, ez, ek = R.batch_pair_multiply(ax[1:], az[1:], np.zeros(P, np.uint8), bx[1:], bz[1:],
                                       np.zeros(P, np.uint8))
    assert np.array_equal(host_cols(x), ex) and np.array_equal(host_cols(z), ez)
    assert np.array_equal(k.cpu().numpy(), ek)


def test_batch_sip(cuda):
    ax, az, _, _ = rng.random_columns(500, 4097, 5)
    bx, bz, _, _ = rng.random_columns(500, 4097, 6)
    got = pl.batch_sip(planes(ax, cuda), planes(az, cuda), planes(bx, cuda), planes(bz, cuda))
    assert np.array_equal(got.cpu().numpy(), R.sip(ax, az, bx, bz).astype(np.uint8))


def test_single_string_known_answers(cuda):
    P = pl.ps_from_label
    # SPEC.md:65 / PAPER.md:179  XZ = -iY
    assert pl.ps_multiply(P("X"), P("Z")).to_label() == ("Y", 3)
    # SPEC.md:73  ZX = iY
    assert pl.ps_multiply(P("Z"), P("X")).to_label() == ("Y", 1)
    # SPEC.md:82 / PAPER.md:196-202  XIZ * ZIX = YIY (phase: (-i)(i) = 1)
    assert pl.ps_multiply(P("XIZ"), P("ZIX")).to_label() == ("YIY", 0)
    assert pl.ps_commutes(P("XX"), P("ZZ")) and not pl.ps_commutes(P("XI"), P("ZI"))
    assert pl.symplectic_inner_product(P("XIZ"), P("ZIX")) == 0
    with pytest.raises(pl.DimensionError):
        pl.ps_multiply(P("X"), P("XX"))


def test_single_qubit_table(cuda):
    """The 16-entry single-qubit product table against dense matrices."""
    mats = {"I": np.eye(2), "X": np.array([[0, 1], [1, 0]]), "Y": np.array([[0, -1j], [1j, 0]]),
            "Z": np.array([[1, 0], [0, -1]])}
    for a in "IXYZ":
        for b in "IXYZ":
            lab, k = pl.ps_multiply(pl.ps_from_label(a), pl.ps_from_label(b)).to_label()
            assert np.allclose(mats[a] @ mats[b], (1j ** k) * mats[lab])


def test_dense_oracle_random_pairs(cuda):
    """Kronecker-product oracle on random n<=4 pairs."""
    mats = {0: np.eye(2), 1: np.array([[0, 1], [1, 0]]), 2: np.array([[1, 0], [0, -1]]),
            3: np.array([[0, -1j], [1j, 0]])}
    r = np.random.default_rng(0)
    for _ in range(60):
        n = int(r.integers(1, 5))
        la = "".join(r.choice(list("IXYZ"), n))
        lb = "".join(r.choice(list("IXYZ"), n))
        ka, kb = int(r.integers(4)), int(r.integers(4))
        pa, pb = pl.ps_from_label(la, ka), pl.ps_from_label(lb, kb)

        def dense(p):
            m = np.array([[1.0 + 0j]])
            for ch in p.label:
                m = np.kron(m, mats["IXZY".index(ch)])
            return (1j ** p.phase) * m

        assert np.allclose(dense(pa) @ dense(pb), dense(pl.ps_multiply(pa, pb)))
        comm = np.allclose(dense(pa) @ dense(pb), dense(pb) @ dense(pa))
        assert pl.ps_commutes(pa, pb) == comm


@pytest.mark.parametrize("n", [500, 64])
def test_outer_raw_golden(cuda, n):
    g = golden(f"outer_raw_n{n}")
    a = pl.PauliSumSoA.from_columns(n, g["ax"], g["az"], g["af"], g["ac"], device=cuda)
    b = pl.PauliSumSoA.from_columns(n, g["bx"], g["bz"], g["bf"], g["bc"], device=cuda)
    out = pl.sum_multiply(a, b, combine=False)
    x, z, k, c = out.columns()
    assert np.array_equal(x, g["ox"]) and np.array_equal(z, g["oz"]) and np.array_equal(k, g["ok"])
    assert np.array_equal(c, g["oc"])  # numpy's FMA complex product, bit for bit


def test_outer_raw_config2_shape(cuda):
    (a, b) = rng.config_columns(2, scale=0.3)
    A = pl.PauliSumSoA.from_columns(500, *a, device=cuda)
    B = pl.PauliSumSoA.from_columns(500, *b, device=cuda)
    x, z, k, c = pl.sum_multiply(A, B, combine=False).columns()
    ex, ez, ek, ec = R.outer_raw(*a, *b)
    assert np.array_equal(x, ex) and np.array_equal(z, ez) and np.array_equal(k, ek)
    np.testing.assert_allclose(c, ec, rtol=1e-15, atol=0)
