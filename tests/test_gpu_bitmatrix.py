"""GPU parity: K5 commutation bitmatrix (both methods) vs the reference/oracle."""

import numpy as np
import torch
import pytest

from conftest import golden
from oracle import numpy_ref as R
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["bitmatrix_c5", "bitmatrix_dense100"])
@pytest.mark.parametrize("method", ["lists", "direct", "tensor", "auto"])
def test_bitmatrix_golden(cuda, name, method):
    g = golden(name)
    m = g["x"].shape[0]
    n = 500 if g["x"].shape[1] == 8 else 100
    s = pl.PauliSumSoA.from_columns(n, g["x"], g["z"], np.zeros(m, np.uint8),
                                    np.ones(m, np.complex128), device=cuda)
    words = pl.commutation_bitmatrix(s, method=method)
    bits = pl.unpack_bits(words, m).cpu().numpy()
    assert np.array_equal(bits, g["bits"])
    assert np.array_equal(words.cpu().numpy().view(np.uint32), R.pack_bitrows(g["bits"]))


@pytest.mark.parametrize("method", ["lists", "direct", "tensor", "auto"])
@pytest.mark.parametrize("W,n", [(1, 50), (2, 100), (4, 256), (8, 500), (16, 1000)])
def test_bitmatrix_blocks_all_tiers(cuda, method, W, n):
    if W == 16 and method in ("lists", "tensor"):
        pytest.skip("lists and tensor methods cover W <= 8")
    m = 2500
    x, z, _, _ = rng.random_columns(n, m, 31 + W)
    # sparsify half the rows so both sparse and dense rows occur
    mask = rng.local_columns(n, m, rng.SplitMix64(3), n, (1, 6))
    x[::2], z[::2] = mask[0][::2], mask[1][::2]
    s = pl.PauliSumSoA.from_columns(n, x, z, np.zeros(m, np.uint8), np.ones(m, np.complex128),
                                    device=cuda)
    for (r0, rows, c0, cols) in [(0, m, 0, m), (17, 1000, 64, 1500), (m - 3, 3, 1024, 1476),
                                 (5, 300, 2048, 452)]:
        words = pl.commutation_bitmatrix(s, row0=r0, rows=rows, col0=c0, cols=cols, method=method)
        got = pl.unpack_bits(words, cols).cpu().numpy()
        exp = R.bitmatrix(x, z, r0, r0 + rows, c0, c0 + cols)
        assert np.array_equal(got, exp), (r0, rows, c0, cols)
        # trailing bits of the last word are zero
        tail = cols % 32
        if tail:
            last = words[:, -1].cpu().numpy().view(np.uint32)
            assert not (last >> np.uint32(tail)).any()


def test_bitmatrix_config5_row_sample(cuda):
    """Config-5 input (scaled); sampled row blocks vs the oracle."""
    x, z, f, c = rng.c5_columns(20000, seed=4)
    s = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=cuda)
    words = pl.commutation_bitmatrix(s)
    assert tuple(words.shape) == (20000, 625)
    for r0 in (0, 9999, 19936):
        got = pl.unpack_bits(words[r0:r0 + 64], 20000).cpu().numpy()
        assert np.array_equal(got, R.bitmatrix(x, z, r0, r0 + 64, 0, 20000))
    # symmetry of the full matrix
    full = pl.unpack_bits(words[:2048], 20000)[:, :2048].cpu().numpy()
    assert np.array_equal(full, full.T)


@pytest.mark.parametrize("n", [64, 100, 200, 500])
def test_bitmatrix_tensor_dense_auto(cuda, n):
    """Dense rows (uniform random strings): 'auto' takes the tcgen05 int8 path;
    every method agrees bit for bit, sampled rows match the oracle."""
    m = 3000
    x, z, _, _ = rng.random_columns(n, m, 77)
    s = pl.PauliSumSoA.from_columns(n, x, z, np.zeros(m, np.uint8), np.ones(m, np.complex128),
                                    device=cuda)
    words = {meth: pl.commutation_bitmatrix(s, method=meth) for meth in ("auto", "tensor", "direct")}
    assert torch.equal(words["auto"], words["tensor"]) and torch.equal(words["tensor"], words["direct"])
    for r in (0, 127, 128, 1500, m - 1):
        exp = R.pack_bitrows(R.bitmatrix(x, z, r, r + 1, 0, m))
        assert np.array_equal(words["tensor"][r:r + 1].cpu().numpy().view(np.uint32), exp)
