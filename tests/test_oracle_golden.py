"""CPU: pin the oracle (numpy + C restatements) to the reference's golden outputs."""

import numpy as np
import pytest

from conftest import golden
from oracle import cgreedy, numpy_ref as R


@pytest.mark.parametrize("n", [40, 100, 200, 500, 1000])
def test_batch_multiply_oracle(n):
    g = golden(f"batch_n{n}")
    x, z, k = R.batch_pair_multiply(g["ax"], g["az"], g["af"], g["bx"], g["bz"], g["bf"])
    assert np.array_equal(x, g["ox"]) and np.array_equal(z, g["oz"]) and np.array_equal(k, g["ok"])


@pytest.mark.parametrize("n", [500, 64])
def test_outer_raw_oracle(n):
    g = golden(f"outer_raw_n{n}")
    for threads in (1, 3):
        x, z, k, c = R.outer_raw(g["ax"], g["az"], g["af"], g["ac"], g["bx"], g["bz"], g["bf"],
                                 g["bc"], threads=threads)
        assert np.array_equal(x, g["ox"]) and np.array_equal(z, g["oz"])
        assert np.array_equal(k, g["ok"])
        np.testing.assert_allclose(c, g["oc"], rtol=1e-15, atol=0)


def _check_combined(got, g, tol=1e-12):
    x, z, k, c = got
    assert np.array_equal(x, g["ox"]) and np.array_equal(z, g["oz"])
    assert not k.any() and not g["ok"].any()
    scale = max(np.abs(g["oc"]).sum(), 1e-300)
    assert np.abs(c - g["oc"]).max(initial=0.0) <= tol * scale


def test_outer_combine_oracle():
    g = golden("outer_c2")
    _check_combined(R.outer_combine(g["ax"], g["az"], g["af"], g["ac"], g["bx"], g["bz"],
                                    g["bf"], g["bc"]), g)


def test_outer_hh_oracle():
    g = golden("outer_hh")
    h = (g["hx"], g["hz"], g["hf"], g["hc"])
    _check_combined(R.outer_combine(*h, *h), g)


def test_simplify_oracle():
    g = golden("simplify_c5")
    _check_combined(R.combine(g["x"], g["z"], g["f"], g["c"]), g)


GROUP_CASES = ["rand6_s1", "rand6_s2", "rand6_s3", "jw2000", "sparse500", "dense500", "allz"]


@pytest.mark.parametrize("name", GROUP_CASES)
def test_greedy_oracle_c(name):
    g = golden(f"group_{name}")
    gof, ng, pc = cgreedy.greedy(g["x"], g["z"])
    assert np.array_equal(gof, g["group_of"])
    assert ng == int(g["n_groups"]) and pc == int(g["pair_checks"])
    assert R.pair_checks_from_assignment(gof) == pc


@pytest.mark.parametrize("name", ["rand6_s1", "rand6_s2", "sparse500", "allz"])
def test_greedy_oracle_numpy(name):
    g = golden(f"group_{name}")
    groups, pc = R.greedy(g["x"], g["z"])
    gof = np.zeros(g["x"].shape[0], np.int32)
    for gi, grp in enumerate(groups):
        gof[grp] = gi
    assert np.array_equal(gof, g["group_of"]) and pc == int(g["pair_checks"])


def test_allz_one_group():
    g = golden("group_allz")
    assert int(g["n_groups"]) == 1


@pytest.mark.parametrize("name", ["bitmatrix_c5", "bitmatrix_dense100"])
def test_bitmatrix_oracle(name):
    g = golden(name)
    m = g["x"].shape[0]
    bits = R.bitmatrix(g["x"], g["z"], 0, m, 0, m)
    assert np.array_equal(bits, g["bits"])
    packed = R.pack_bitrows(bits)
    assert packed.shape == (m, (m + 31) // 32)
    # unpack round trip
    un = np.unpackbits(packed.view(np.uint8), axis=1, bitorder="little")[:, :m]
    assert np.array_equal(un, bits)
