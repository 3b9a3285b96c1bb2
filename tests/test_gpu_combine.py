"""GPU parity: outer product + merge (K2-K4) and sort_and_combine vs reference/oracle.

Contract (north star): merged X/Z bits, phases (all 0) and key sets bit-exact;
coefficients within 1e-12 relative to the summed magnitudes.
"""

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import numpy_ref as R
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng

pytestmark = pytest.mark.gpu

TOL = 1e-12


def check_combined(out, exp):
    x, z, k, c = out.columns() if hasattr(out, "columns") else out
    ex, ez, ek, ec = exp
    assert x.shape == ex.shape, (x.shape, ex.shape)
    assert np.array_equal(x, ex) and np.array_equal(z, ez)
    assert not np.asarray(k).any() and not np.asarray(ek).any()
    scale = max(float(np.abs(ec).sum()), 1e-300)
    err = float(np.abs(np.asarray(c) - ec).max(initial=0.0))
    assert err <= TOL * scale, (err, scale)


def soa(n, cols, dev):
    return pl.PauliSumSoA.from_columns(n, *cols, device=dev)


def test_outer_c2_golden(cuda):
    g = golden("outer_c2")
    a = soa(500, (g["ax"], g["az"], g["af"], g["ac"]), cuda)
    b = soa(500, (g["bx"], g["bz"], g["bf"], g["bc"]), cuda)
    check_combined(pl.sum_multiply(a, b), (g["ox"], g["oz"], g["ok"], g["oc"]))


def test_outer_hh_golden(cuda):
    g = golden("outer_hh")
    h = soa(64, (g["hx"], g["hz"], g["hf"], g["hc"]), cuda)
    check_combined(h * h, (g["ox"], g["oz"], g["ok"], g["oc"]))


def test_simplify_golden(cuda):
    g = golden("simplify_c5")
    s = soa(500, (g["x"], g["z"], g["f"], g["c"]), cuda)
    check_combined(pl.sort_and_combine(s), (g["ox"], g["oz"], g["ok"], g["oc"]))


def test_config2_full(cuda):
    """Config 2 at full size (10^6 pair products) vs the oracle."""
    a, b = rng.config_columns(2)
    out = pl.sum_multiply(soa(500, a, cuda), soa(500, b, cuda))
    check_combined(out, R.outer_combine(*a, *b))


def test_config4_scaled(cuda):
    """Config 4 shape at 1500 x 1500 (2.25e6 products, 96-bit keys, level-2 split)."""
    a, b = rng.config_columns(4, scale=0.15)
    out = pl.sum_multiply(soa(500, a, cuda), soa(500, b, cuda))
    check_combined(out, R.outer_combine(*a, *b))


def test_config5_simplify_scaled(cuda):
    """Config 5 shape (full-width 1000-bit keys, 10% duplicates) at 200k terms."""
    x, z, f, c = rng.c5_columns(200_000, seed=4)
    f = np.random.default_rng(3).integers(0, 4, x.shape[0]).astype(np.uint8)
    out = pl.sort_and_combine(soa(500, (x, z, f, c), cuda))
    check_combined(out, R.combine(x, z, f, c))


def test_dense_random_keys(cuda):
    """Uniform random 500-qubit strings: every key bit used (KW=16)."""
    a = rng.random_columns(500, 300, 1)
    b = rng.random_columns(500, 200, 2)
    out = pl.sum_multiply(soa(500, a, cuda), soa(500, b, cuda))
    check_combined(out, R.outer_combine(*a, *b))


@pytest.mark.parametrize("n", [1, 64, 100, 256, 1000])
def test_tiers_hh(cuda, n):
    h = rng.local_columns(n, 700, rng.SplitMix64(n), min(n, 12), (1, min(n, 4)))
    s = soa(n, h, cuda)
    check_combined(s * s, R.outer_combine(*h, *h))
    check_combined(s.sort_and_combine(), R.combine(*h))


def test_runs_longer_than_leaf(cuda):
    """9000 copies of X (random coefficients and phases) times {X, Y, Z}: three
    keys each repeated 9000 times (> the 8192-item shared-memory leaf), which
    no splitter can divide, exercising the in-place global-memory leaf path."""
    r = np.random.default_rng(9)
    m = 9000
    a = (np.ones((m, 1), np.uint64), np.zeros((m, 1), np.uint64),
         r.integers(0, 4, m).astype(np.uint8), r.normal(size=m) + 1j * r.normal(size=m))
    b = (np.array([[1], [1], [0]], np.uint64), np.array([[0], [1], [1]], np.uint64),
         np.array([0, 1, 2], np.uint8), np.array([1.0, -0.5j, 2.0], np.complex128))
    out = pl.sum_multiply(soa(3, a, cuda), soa(3, b, cuda))
    check_combined(out, R.outer_combine(*a, *b))
    # the same with the long runs mixed into many distinct keys
    h = rng.local_columns(64, 3000, rng.SplitMix64(77), 40, (1, 3))
    a2 = tuple(np.concatenate([u, v]) for u, v in zip(h, (np.ones((m, 1), np.uint64),
                                                         np.zeros((m, 1), np.uint64), a[2], a[3])))
    out2 = pl.sum_multiply(soa(64, a2, cuda), soa(64, b, cuda))
    check_combined(out2, R.outer_combine(*a2, *b))


def test_eps_and_cancellation(cuda):
    x, z, f, c = rng.c5_columns(5000, seed=1)
    base = pl.sort_and_combine(soa(500, (x, z, f, c), cuda))
    ux, uz, uf, uc = base.columns()
    # a sum with unique keys plus its negation -> empty (SPEC.md:463 (i))
    s = soa(500, (np.concatenate([ux, ux]), np.concatenate([uz, uz]), np.concatenate([uf, uf]),
                  np.concatenate([uc, -uc])), cuda)
    assert len(pl.sort_and_combine(s)) == 0
    # with repeated keys the reference's own summation order decides which
    # runs cancel exactly; the GPU reproduces it (numpy reduceat tree)
    cols = (np.concatenate([x, x]), np.concatenate([z, z]), np.concatenate([f, f]),
            np.concatenate([c, -c]))
    check_combined(pl.sort_and_combine(soa(500, cols, cuda)), R.combine(*cols))
    # shuffled 3x duplication triples the coefficient (ii)
    perm = np.random.default_rng(0).permutation(3 * len(ux))
    s3 = soa(500, tuple(np.concatenate([a] * 3)[perm] for a in (ux, uz, uf, uc)), cuda)
    out3 = pl.sort_and_combine(s3)
    np.testing.assert_allclose(out3.columns()[3], 3 * uc, rtol=1e-14)
    # idempotence bit-exact (iii)
    assert pl.sort_and_combine(base) == base
    # eps drops small terms
    out_e = pl.sort_and_combine(soa(500, (x, z, f, c), cuda), eps=0.5)
    check_combined(out_e, R.combine(x, z, f, c, eps=0.5))
    with pytest.raises(ValueError):
        pl.sort_and_combine(soa(500, (x, z, f, c), cuda), eps=-1.0)


def test_golden_coefficients_bit_exact(cuda):
    """Products use numpy's FMA rounding and runs use numpy's reduceat tree, so
    the merged coefficients equal the reference's bit for bit."""
    g = golden("outer_hh")
    h = soa(64, (g["hx"], g["hz"], g["hf"], g["hc"]), cuda)
    assert np.array_equal((h * h).columns()[3], g["oc"])
    g = golden("simplify_c5")
    s = soa(500, (g["x"], g["z"], g["f"], g["c"]), cuda)
    assert np.array_equal(pl.sort_and_combine(s).columns()[3], g["oc"])
    g = golden("outer_c2")
    a = soa(500, (g["ax"], g["az"], g["af"], g["ac"]), cuda)
    b = soa(500, (g["bx"], g["bz"], g["bf"], g["bc"]), cuda)
    assert np.array_equal((a * b).columns()[3], g["oc"])
    g = golden("outer_raw_n500")
    a = soa(500, (g["ax"], g["az"], g["af"], g["ac"]), cuda)
    b = soa(500, (g["bx"], g["bz"], g["bf"], g["bc"]), cuda)
    assert np.array_equal(pl.sum_multiply(a, b, combine=False).columns()[3], g["oc"])


def test_empty_and_single(cuda):
    e = pl.PauliSumSoA.empty(500, device=cuda)
    one = pl.PauliSumSoA.from_terms([(2.0, "XYZ" + "I" * 497)], device=cuda)
    assert len(e * one) == 0 and len(one * e) == 0 and len(e.sort_and_combine()) == 0
    sq = one * one
    x, z, k, c = sq.columns()
    assert len(sq) == 1 and not x.any() and not z.any() and c[0] == 4.0


def test_determinism_and_host_path(cuda):
    a, b = rng.config_columns(2, scale=0.5)
    A, B = soa(500, a, cuda), soa(500, b, cuda)
    r1 = pl.sum_multiply(A, B)
    r2 = pl.sum_multiply(A, B, threads=8)
    assert r1 == r2
    # host sums in -> host sum out, identical result (end-to-end path)
    h = pl.sum_multiply(A.cpu(), B.cpu())
    assert h.device.type == "cpu" and h == r1.cpu()
    # AoS drop-in
    aos = pl.PauliSum.from_columns(500, *a).multiply(pl.PauliSum.from_columns(500, *b))
    assert isinstance(aos, pl.PauliSum) and len(aos) == len(r1)


def test_host_path_zero_planes_on_dirty_buffers(cuda):
    """Host results: planes proved zero by the plan are cleared on the host,
    not copied.  Recycled pinned buffers hold stale data (a dense result
    first), so a missed clear would show; sort_and_combine shares the path."""
    from paper_2605_25974_b200 import sums as S
    ax, az, af, ac = rng.random_columns(500, 300, 7)
    dense = pl.PauliSumSoA.from_columns(500, ax, az, af, ac)          # every plane nonzero
    sparse_a, sparse_b = rng.config_columns(2, scale=0.3)              # qubits 0..23 only
    A, B = soa(500, sparse_a, None), soa(500, sparse_b, None)
    for _ in range(2):
        d = pl.sort_and_combine(dense)                                 # dirties the pinned pool
        assert S.LAST_D2H_BYTES == d.payload_nbytes - len(d)           # only the phase bytes skipped
        del d
        h = pl.sum_multiply(A, B)
        assert h.device.type == "cpu"
        m = len(h)
        # x0, z0 and the coefficients, plus however many of the 14 proved-zero
        # planes the DMA engine took while the host cleared the others
        extra = S.LAST_D2H_BYTES - m * (2 * 8 + 16)
        assert 0 <= extra <= 14 * 8 * m
        ref = pl.sum_multiply(A.cuda(), B.cuda()).cpu()
        assert h == ref
        assert not h.x[1:].any() and not h.z[1:].any() and not h.flags.any()
        hs = pl.sort_and_combine(pl.sum_multiply(A, B, combine=False))
        assert hs == ref
        del h, hs


def test_raw_count_exact(cuda):
    """|output before combine| = |a|*|b| exactly."""
    a, b = rng.config_columns(2, scale=0.05)
    raw = pl.sum_multiply(soa(500, a, cuda), soa(500, b, cuda), combine=False)
    assert len(raw) == 50 * 50


def test_dense_matrix_small(cuda):
    """Outer product equals the dense matrix product at n <= 4."""
    mats = [np.eye(2), np.array([[0, 1], [1, 0]]), np.array([[1, 0], [0, -1]]),
            np.array([[0, -1j], [1j, 0]])]

    def dense(s):
        x, z, k, c = s.columns()
        tot = 0
        for t in range(len(s)):
            m = np.array([[1.0 + 0j]])
            for q in range(s.n):
                code = int((x[t, 0] >> np.uint64(q)) & np.uint64(1)) + 2 * int(
                    (z[t, 0] >> np.uint64(q)) & np.uint64(1))
                m = np.kron(m, mats[code])
            tot = tot + c[t] * (1j ** int(k[t])) * m
        return tot

    r = np.random.default_rng(5)
    for n in (1, 2, 3, 4):
        for _ in range(3):
            la = ["".join(r.choice(list("IXYZ"), n)) for _ in range(int(r.integers(1, 10)))]
            lb = ["".join(r.choice(list("IXYZ"), n)) for _ in range(int(r.integers(1, 10)))]
            A = pl.PauliSumSoA.from_terms([(complex(*r.normal(size=2)), l) for l in la], device=cuda)
            B = pl.PauliSumSoA.from_terms([(complex(*r.normal(size=2)), l) for l in lb], device=cuda)
            assert np.allclose(dense(A) @ dense(B), dense(A * B), atol=1e-12)


def test_buckets_balanced(cuda):
    """Performance guard: the sampled splitters must spread config-4 items over
    the level-1 buckets (a degenerate sample sends everything to one bucket,
    which stays correct but is ~20x slower)."""
    import ctypes as C
    import torch
    from paper_2605_25974_b200 import _native
    from paper_2605_25974_b200._device import ptr, stream_ptr

    a, b = rng.config_columns(4, scale=0.2)
    A, B = soa(500, a, cuda).planes(), soa(500, b, cuda).planes()
    plan = _native.MergePlan()
    _native.call("pl_outer_plan", 8, A.M, B.M, ptr(A.x), ptr(A.z), A.ld, ptr(B.x), ptr(B.z), B.ld,
                 C.byref(plan), stream_ptr(cuda))
    nb = plan.n_buckets
    assert nb > 16
    lib = _native.load()
    send_bytes = A.M * B.M * lib.pl_dist_item_bytes(C.byref(plan))
    ws = torch.empty(lib.pl_dist_workspace_bytes(C.byref(plan), A.M * B.M, nb), dtype=torch.uint8,
                     device=cuda)
    send = torch.empty(send_bytes, dtype=torch.uint8, device=cuda)
    counts = torch.empty(nb, dtype=torch.int32, device=cuda)
    _native.call("pl_outer_partition", C.byref(plan), ptr(A.x), ptr(A.z), ptr(A.k), A.ld, ptr(B.x),
                 ptr(B.z), ptr(B.k), B.ld, 0, B.M, ptr(ws), ws.numel(), ptr(send), ptr(counts),
                 stream_ptr(cuda))
    cnt = counts.cpu().numpy()
    assert cnt.sum() == A.M * B.M
    assert cnt.max() < 4 * cnt.mean(), (cnt.max(), cnt.mean())


def test_sparse_keys_plan_and_parity(cuda):
    """Wide sparse keys (config 5 style) take the set-bit-list key encoding
    (KW 16 -> 4) and still merge exactly; negated duplicates cancel."""
    x, z, f, c = rng.c5_columns(50_000, seed=9)
    x = np.concatenate([x, x[:5000]])
    z = np.concatenate([z, z[:5000]])
    f = np.concatenate([f, f[:5000]])
    c = np.concatenate([c, -c[:5000]])  # exact cancellations
    out = pl.sort_and_combine(soa(500, (x, z, f, c), cuda))
    assert pl.sums.LAST_PLAN["key_words"] < 16
    check_combined(out, R.combine(x, z, f, c))


@pytest.mark.parametrize("n", [200, 1000])
def test_sparse_keys_other_tiers(cuda, n):
    r = np.random.default_rng(n)
    W = pl.words_for(n)
    m = 20_000
    x = np.zeros((m, W), np.uint64)
    z = np.zeros((m, W), np.uint64)
    for t in range(m):  # weight-3 strings, many repeats
        for q in r.choice(n, 3, replace=False) if t % 3 else [1, 2, 3]:
            ltr = r.integers(1, 4)
            if ltr & 1:
                x[t, q // 64] |= np.uint64(1) << np.uint64(q % 64)
            if ltr & 2:
                z[t, q // 64] |= np.uint64(1) << np.uint64(q % 64)
    f = r.integers(0, 4, m).astype(np.uint8)
    c = (r.normal(size=m) + 1j * r.normal(size=m)).astype(np.complex128)
    out = pl.sort_and_combine(soa(n, (x, z, f, c), cuda))
    check_combined(out, R.combine(x, z, f, c))


def test_dense_keys_w16_sort(cuda):
    """n = 1000 uniform random strings: ~1500 set bits per key, dense KW=32 path."""
    x, z, f, c = rng.random_columns(1000, 3000, 5)
    x = np.concatenate([x, x[:100]])
    z = np.concatenate([z, z[:100]])
    f = np.concatenate([f, f[:100]])
    c = np.concatenate([c, c[:100]])
    out = pl.sort_and_combine(soa(1000, (x, z, f, c), cuda))
    check_combined(out, R.combine(x, z, f, c))


def test_leaf_window_ties_fall_back(cuda):
    """Keys that agree on the 24-bit radix window below the leaf's highest
    differing bit but differ further down: the tie segments exceed the
    insertion-sort limit and the leaf takes the bitonic fallback."""
    r = np.random.default_rng(11)
    m = 600
    x = np.zeros((m, 1), np.uint64)
    z = np.zeros((m, 1), np.uint64)
    z[0, 0] = np.uint64(1) << np.uint64(63)  # a different high key bit
    z[1:, 0] = np.uint64(1)                  # shared z part
    x[1:, 0] = r.integers(0, 1 << 20, m - 1).astype(np.uint64)  # low bits differ
    f = r.integers(0, 4, m).astype(np.uint8)
    c = (r.normal(size=m) + 1j * r.normal(size=m)).astype(np.complex128)
    out = pl.sort_and_combine(soa(64, (x, z, f, c), cuda))
    check_combined(out, R.combine(x, z, f, c))


def test_level2_window_ties(cuda):
    """Level 2 classifies on the 32 key bits after the bucket's shared prefix;
    two far-apart clusters whose members differ only 48 bits further down give
    every splitter of a cluster the same window, so every item takes the
    full-key comparison against the tied splitters (and the leaves see long
    shared prefixes)."""
    r = np.random.default_rng(17)
    m = 60_000
    z = np.zeros((m, 1), np.uint64)
    x = np.zeros((m, 1), np.uint64)
    cluster = r.integers(0, 2, m).astype(np.uint64)
    z[:, 0] = (cluster << np.uint64(63)) | r.integers(0, 1 << 16, m).astype(np.uint64)
    f = r.integers(0, 4, m).astype(np.uint8)
    c = (r.normal(size=m) + 1j * r.normal(size=m)).astype(np.complex128)
    out = pl.sort_and_combine(soa(64, (x, z, f, c), cuda))
    assert pl.sums.LAST_PLAN["n_buckets"] > 1 and pl.sums.LAST_PLAN["key_bits"] == 64
    check_combined(out, R.combine(x, z, f, c))


def test_distinct_leaves_with_dropped_terms(cuda):
    """Leaves whose keys are all distinct are written straight from the rank
    order unless a coefficient is dropped: zero operand coefficients (exact
    zero products at eps = 0) and an eps that removes some single-item runs
    send those leaves through the general path; both agree with the oracle."""
    a, b = rng.config_columns(4, scale=0.06)                    # 600 x 600, ~all keys distinct
    ac = a[3].copy()
    ac[::7] = 0.0                                               # exact-zero products
    a0 = (a[0], a[1], a[2], ac)
    out = pl.sum_multiply(soa(500, a0, cuda), soa(500, b, cuda))
    check_combined(out, R.outer_combine(*a0, *b))
    assert len(out) < len(a[0]) * len(b[0])
    eps = 0.3
    out = pl.sum_multiply(soa(500, a, cuda), soa(500, b, cuda), eps=eps)
    exp = R.outer_combine(*a, *b, eps=eps)
    check_combined(out, exp)
    assert 0 < len(out) < len(a[0]) * len(b[0])
    keep_all = pl.sum_multiply(soa(500, a0, cuda), soa(500, b, cuda), eps=-1.0)
    assert len(keep_all) == len(R.outer_combine(*a0, *b, eps=-1.0)[3])


def test_eps_drop_large(cuda):
    """eps drops on a 10^6-product outer product (strict > eps keeps)."""
    a, b = rng.config_columns(2)
    eps = 0.5
    out = pl.sum_multiply(soa(500, a, cuda), soa(500, b, cuda), eps=eps)
    exp = R.outer_combine(*a, *b, eps=eps)
    check_combined(out, exp)


def test_sparse_keys_oversized_run(cuda):
    """One sparse key repeated 3000 times (longer than a leaf) among config-5
    terms: the in-place global-memory leaf path with set-bit-list keys."""
    x, z, f, c = rng.c5_columns(20_000, seed=21)
    rep = 3000
    x = np.concatenate([x, np.repeat(x[7:8], rep, axis=0)])
    z = np.concatenate([z, np.repeat(z[7:8], rep, axis=0)])
    f = np.concatenate([f, np.full(rep, 1, np.uint8)])
    r = np.random.default_rng(5)
    c = np.concatenate([c, (r.normal(size=rep) + 1j * r.normal(size=rep))])
    out = pl.sort_and_combine(soa(500, (x, z, f, c), cuda))
    assert pl.sums.LAST_PLAN["key_words"] < 16
    check_combined(out, R.combine(x, z, f, c))


@pytest.mark.parametrize("m", [0, 1, 2, 33])
def test_tiny_sums(cuda, m):
    x, z, f, c = rng.c5_columns(max(m, 1), seed=3)
    x, z, f, c = x[:m], z[:m], f[:m], c[:m]
    out = pl.sort_and_combine(soa(500, (x, z, f, c), cuda))
    if m == 0:
        assert len(out) == 0
    else:
        check_combined(out, R.combine(x, z, f, c))


def test_sampler_constant_leading_key_word(cuda):
    """Every term shares its letters on qubits 0..63 (packed key word 0 is the
    same for all terms): the level-1 sampler's word-0 composites all tie and it
    must fall back to its full-key sort; result still equals the oracle."""
    n, m = 300, 40_000
    x, z, f, c = rng.random_columns(n, m, 91)
    x[:, 0] = x[0, 0]
    z[:, 0] = z[0, 0]
    f = (np.arange(m) % 4).astype(np.uint8)
    x = np.concatenate([x, x[:5000]])
    z = np.concatenate([z, z[:5000]])
    f = np.concatenate([f, f[:5000]])
    c = np.concatenate([c, -c[:5000]])
    got = pl.sort_and_combine(soa(n, (x, z, f, c), cuda))
    ex, ez, ek, ec = R.combine(x, z, f, c)
    gx, gz, gk, gc = got.columns()
    assert np.array_equal(gx, ex) and np.array_equal(gz, ez)
    assert np.abs(gc - ec).max(initial=0) <= 1e-12 * np.abs(ec).sum()


def test_two_phase_exact_emit_equals_single_call(cuda, monkeypatch):
    """Large merges run as merge + count, then pl_merge_emit into exactly sized
    planes; forcing that path on small inputs gives the same sums."""
    a, b = rng.config_columns(2, 0.3)
    A, B = soa(500, a, cuda), soa(500, b, cuda)
    h = rng.local_columns(64, 800, rng.SplitMix64(3), 12, (1, 3))
    H = soa(64, h, cuda)
    x, z, f, c = rng.c5_columns(20_000, seed=9)
    S = soa(500, (x, z, f, c), cuda)
    ref = [pl.outer_multiply(A, B), H * H, pl.sort_and_combine(S)]
    monkeypatch.setattr(pl.sums, "_TWO_PHASE_MIN", 0)
    got = [pl.outer_multiply(A, B), H * H, pl.sort_and_combine(S)]
    for r, g in zip(ref, got):
        assert g == r
        assert g.x.shape[1] == len(g)  # exactly sized planes
