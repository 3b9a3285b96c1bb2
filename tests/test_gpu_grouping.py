"""GPU parity: K6 greedy grouping — group assignment and pair_checks bit-exact
with the reference (golden) and the C restatement (oracle/greedy.c)."""

import numpy as np
import pytest

from conftest import golden
from oracle import cgreedy, numpy_ref as R
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng

pytestmark = pytest.mark.gpu

CASES = ["rand6_s1", "rand6_s2", "rand6_s3", "jw2000", "sparse500", "dense500", "allz"]


def soa(n, x, z, dev):
    m = x.shape[0]
    return pl.PauliSumSoA.from_columns(n, x, z, np.zeros(m, np.uint8), np.ones(m, np.complex128),
                                       device=dev)


@pytest.mark.parametrize("name", CASES)
def test_grouping_golden(cuda, name):
    g = golden(f"group_{name}")
    s = soa(int(g["n"]), g["x"], g["z"], cuda)
    gof, ng, pc = pl.group_assignment(s)
    assert np.array_equal(gof.cpu().numpy(), g["group_of"])
    assert int(ng.item()) == int(g["n_groups"]) and int(pc.item()) == int(g["pair_checks"])
    # reference API surface
    stats = pl.GroupingStats()
    part = pl.group_greedy(s, stats=stats)
    assert stats.pair_checks == int(g["pair_checks"]) and part.group_count() == int(g["n_groups"])
    assert all(grp == sorted(grp) for grp in part.groups)
    assert pl.validate_partition(s, part).ok


def check_vs_oracle(n, x, z, dev):
    gof, ng, pc = pl.group_assignment(soa(n, x, z, dev))
    eg, eng, epc = cgreedy.greedy(x, z)
    got = gof.cpu().numpy()
    if not np.array_equal(got, eg):
        bad = int(np.flatnonzero(got != eg)[0])
        raise AssertionError(f"first mismatch at term {bad}: {got[bad]} vs {eg[bad]}")
    assert int(ng.item()) == eng and int(pc.item()) == epc


@pytest.mark.parametrize("m", [1, 2, 1023, 1024, 1025, 5000])
def test_batch_boundaries(cuda, m):
    x, z, _, _ = rng.local_columns(100, m, rng.SplitMix64(m), 100, (1, 6))
    check_vs_oracle(100, x, z, cuda)


@pytest.mark.parametrize("W,n", [(1, 40), (2, 100), (4, 200), (8, 500), (16, 1000)])
def test_tiers(cuda, W, n):
    x, z, _, _ = rng.local_columns(n, 3000, rng.SplitMix64(W), n, (1, 8))
    check_vs_oracle(n, x, z, cuda)


def test_dense_random(cuda):
    x, z, _, _ = rng.random_columns(64, 4000, 3)
    check_vs_oracle(64, x, z, cuda)


def test_config3_prefix(cuda):
    """Config 3 (JW-style, n=100): a 30k-term prefix (prefix-closed, so it equals
    the first 30k assignments of the full run)."""
    x, z, _, _ = rng.config_columns(3, scale=0.3)
    check_vs_oracle(100, x, z, cuda)


def test_config5_prefix(cuda):
    x, z, _, _ = rng.c5_columns(1_000_000, seed=4)
    check_vs_oracle(500, x[:8000], z[:8000], cuda)


def test_all_commuting_one_group(cuda):
    r = np.random.default_rng(0)
    z = r.integers(0, 2 ** 62, size=(3000, 2)).astype(np.uint64)
    z[:, 1] &= np.uint64((1 << 36) - 1)
    x = np.zeros_like(z)
    gof, ng, pc = pl.group_assignment(soa(100, x, z, cuda))
    assert int(ng.item()) == 1 and int(pc.item()) == 3000 * 2999 // 2
    assert int(pc.item()) <= 3000 ** 2


@pytest.mark.slow
def test_config3_full(cuda):
    x, z, _, _ = rng.config_columns(3)
    check_vs_oracle(100, x, z, cuda)


# ------------------------------------------------------------ f3 parallel grouping
@pytest.mark.parametrize("name", ["group_par_rand", "group_par_dense", "group_par_jw"])
@pytest.mark.parametrize("chunks", [1, 2, 5, 16])
def test_group_greedy_parallel_golden(cuda, name, chunks):
    g = golden(name)
    n = int(g["n"])
    m = g["x"].shape[0]
    s = pl.PauliSumSoA.from_columns(n, g["x"], g["z"], np.zeros(m, np.uint8),
                                    np.ones(m, np.complex128), device=cuda)
    st = pl.GroupingStats()
    part = pl.group_greedy_parallel(s, chunks, stats=st)
    flat = [t for grp in part.groups for t in grp]
    assert np.array_equal(flat, g[f"members{chunks}"])
    assert np.array_equal(np.cumsum([0] + [len(x) for x in part.groups]), g[f"offsets{chunks}"])
    assert st.pair_checks == int(g[f"checks{chunks}"])
    assert pl.validate_partition(s, part).ok


def test_group_greedy_parallel_one_chunk_equals_greedy(cuda):
    x, z, f, c = rng.config_columns(3, scale=0.05)
    s = pl.PauliSumSoA.from_columns(100, x, z, f, c, device=cuda)
    assert pl.group_greedy_parallel(s, 1).groups == pl.group_greedy(s).groups


def test_group_greedy_parallel_matches_oracle_c3_prefix(cuda):
    x, z, f, c = rng.config_columns(3, scale=0.1)
    s = pl.PauliSumSoA.from_columns(100, x, z, f, c, device=cuda)
    st = pl.GroupingStats()
    part = pl.group_greedy_parallel(s, 8, stats=st)
    groups, checks = R.greedy_parallel(x, z, 8)
    assert part.groups == groups and st.pair_checks == checks


def test_group_greedy_parallel_errors(cuda):
    s = pl.PauliSumSoA.from_columns(10, *rng.random_columns(10, 4, 1), device=cuda)
    with pytest.raises(ValueError):
        pl.group_greedy_parallel(s, 0)


@pytest.mark.parametrize("cap", ["0", "37"])
def test_deep_fit_queue_overflow_falls_back_inline(cuda, cap, monkeypatch):
    """(term, group) pairs that do not fit the deep-fit queue are finished by
    the owning warp inside k_group_fit: same assignment and pair_checks with an
    empty or a tiny queue (config 3 prefix: groups of many chunks)."""
    from oracle import cgreedy

    x, z, f, c = rng.config_columns(3, scale=0.2)
    gof_ref, ng_ref, pc_ref = cgreedy.greedy(x, z)
    monkeypatch.setenv("PLB_DEEP_QUEUE_CAP", cap)
    S = pl.PauliSumSoA.from_columns(100, x, z, f, c, device=cuda)
    gof, ng, pc = pl.group_assignment(S)
    assert np.array_equal(gof.cpu().numpy(), np.asarray(gof_ref))
    assert int(ng.item()) == ng_ref and int(pc.item()) == pc_ref
