"""GPU: the K7 multi-GPU stages, emulated on one device (virtual ranks run
sequentially, exchange by slicing): the rank-order concatenation of the shards
is bit-identical to the single-GPU merge for every rank count."""

import numpy as np
import pytest

import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import dist as pdist, rng
from oracle import numpy_ref as R

pytestmark = pytest.mark.gpu


def soa(n, cols, dev):
    return pl.PauliSumSoA.from_columns(n, *cols, device=dev)


@pytest.mark.parametrize("cfg,scale", [(2, 1.0), (4, 0.08)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sharded_equals_single(cuda, cfg, scale, world):
    a, b = rng.config_columns(cfg, scale)
    A, B = soa(500, a, cuda), soa(500, b, cuda)
    single = pl.outer_multiply(A, B)
    shards = pdist.emulate_sharded(A, B, world)
    assert pdist.concat(shards) == single


def test_sharded_hh_cancellation(cuda):
    h = rng.local_columns(64, 800, rng.SplitMix64(3), 12, (1, 3))
    H = soa(64, h, cuda)
    single = H * H
    assert pdist.concat(pdist.emulate_sharded(H, H, 4)) == single
    ex = R.outer_combine(*h, *h)
    assert np.array_equal(single.columns()[0], ex[0])


def test_sharded_api_single_process(cuda):
    """sharded_outer_multiply without a process group = the single-GPU call."""
    a, b = rng.config_columns(2, 0.3)
    A, B = soa(500, a, cuda), soa(500, b, cuda)
    assert pdist.sharded_outer_multiply(A, B) == pl.outer_multiply(A, B)
    words, (r0, r1) = pdist.sharded_bitmatrix(A)
    assert (r0, r1) == (0, len(A)) and words.shape[0] == len(A)
