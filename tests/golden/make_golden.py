"""Generate golden fixtures by RUNNING THE REFERENCE (paulialg, pure numpy).

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Each fixture stores the inputs and the reference's outputs so the oracle and
the GPU kernels can be checked on any machine without /root/reference.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import paulialg as ref  # noqa: E402
from paulialg import bench as ref_bench  # noqa: E402
from paulialg import strings as ref_strings  # noqa: E402
from paulialg.sums import PauliSum as RefSum  # noqa: E402

from paper_2605_25974_b200 import rng  # noqa: E402


def ref_sum(n, x, z, f, c):
    return RefSum._from_columns(n, np.ascontiguousarray(x), np.ascontiguousarray(z),
                                np.asarray(f, np.uint8), np.asarray(c, np.complex128))


def cols(s):
    x, z, f, c = s._columns()
    return (np.ascontiguousarray(x), np.ascontiguousarray(z), np.asarray(f).copy(),
            np.asarray(c).copy())


def save(name, **arrs):
    np.savez_compressed(HERE / f"{name}.npz", **arrs)
    print(name, {k: v.shape for k, v in arrs.items()})


def main():
    r = np.random.default_rng(20261020)

    # 1. generator pin: config-1 draws equal the reference random_sum
    for n, m, seed in ((500, 256, 0), (100, 64, 7)):
        s = ref.random_sum(n, m, seed)
        x, z, f, c = cols(s)
        save(f"rng_n{n}_s{seed}", x=x, z=z, f=f, c=c)

    # 2. batched pair multiply (bench.py:168-177) at every tier
    for n, P in ((40, 333), (100, 257), (200, 129), (500, 300), (1000, 65)):
        a = ref.random_sum(n, P, 11)
        b = ref.random_sum(n, P, 12)
        ax, az, _, _ = cols(a)
        bx, bz, _, _ = cols(b)
        af = r.integers(0, 4, P).astype(np.uint8)
        bf = r.integers(0, 4, P).astype(np.uint8)
        ox, oz, ok = ref_bench._batch_pair_multiply(ax, az, af, bx, bz, bf)
        save(f"batch_n{n}", ax=ax, az=az, af=af, bx=bx, bz=bz, bf=bf, ox=ox, oz=oz, ok=ok)

    # 3. raw outer product (sums.py:144-174), random phases and complex coeffs
    for n, ma, mb in ((500, 17, 23), (64, 40, 9)):
        ax, az, _, _ = cols(ref.random_sum(n, ma, 21))
        bx, bz, _, _ = cols(ref.random_sum(n, mb, 22))
        af = r.integers(0, 4, ma).astype(np.uint8)
        bf = r.integers(0, 4, mb).astype(np.uint8)
        ac = r.normal(size=ma) + 1j * r.normal(size=ma)
        bc = r.normal(size=mb) + 1j * r.normal(size=mb)
        out = ref.sum_multiply(ref_sum(n, ax, az, af, ac), ref_sum(n, bx, bz, bf, bc), combine=False)
        ox, oz, ok, oc = cols(out)
        save(f"outer_raw_n{n}", ax=ax, az=az, af=af, ac=ac, bx=bx, bz=bz, bf=bf, bc=bc,
             ox=ox, oz=oz, ok=ok, oc=oc)

    # 4. outer product + combine: config-2 shape (4-local on 24 qubits) at 120x150
    st = rng.SplitMix64(1)
    a = rng.local_columns(500, 120, st, 24, 4)
    b = rng.local_columns(500, 150, st, 24, 4)
    af = r.integers(0, 4, 120).astype(np.uint8)
    out = ref.sum_multiply(ref_sum(500, a[0], a[1], af, a[3]), ref_sum(500, *b))
    ox, oz, ok, oc = cols(out)
    save("outer_c2", ax=a[0], az=a[1], af=af, ac=a[3], bx=b[0], bz=b[1], bf=b[2], bc=b[3],
         ox=ox, oz=oz, ok=ok, oc=oc)

    # 5. H*H: exact cancellations and the identity run (length |H|)
    h = rng.local_columns(64, 60, rng.SplitMix64(5), 10, 3)
    out = ref.sum_multiply(ref_sum(64, *h), ref_sum(64, *h))
    ox, oz, ok, oc = cols(out)
    save("outer_hh", hx=h[0], hz=h[1], hf=h[2], hc=h[3], ox=ox, oz=oz, ok=ok, oc=oc)

    # 6. sort_and_combine: config-5 shape (weight 2..12 / 500 qubits, 10% dups)
    x, z, f, c = rng.c5_columns(3000, seed=9)
    f = r.integers(0, 4, 3000).astype(np.uint8)
    # add exact negations of 50 terms (cancel to zero) and triple 20 terms
    neg = r.choice(3000, 50, replace=False)
    tri = r.choice(3000, 20, replace=False)
    x = np.concatenate([x, x[neg], x[tri], x[tri]])
    z = np.concatenate([z, z[neg], z[tri], z[tri]])
    f2 = np.concatenate([f, f[neg], f[tri], f[tri]])
    c = np.concatenate([c, -c[neg], c[tri], c[tri]])
    perm = r.permutation(x.shape[0])
    x, z, f2, c = x[perm], z[perm], f2[perm], c[perm]
    out = ref.sort_and_combine(ref_sum(500, x, z, f2, c))
    ox, oz, ok, oc = cols(out)
    save("simplify_c5", x=x, z=z, f=f2, c=c, ox=ox, oz=oz, ok=ok, oc=oc)

    # 7. greedy grouping + pair_checks (grouping.py:67-95)
    cases = {}
    for seed in (1, 2, 3):
        cases[f"rand6_s{seed}"] = (6,) + cols(ref.random_sum(6, 64, seed))[:2]
    cases["jw2000"] = (100,) + rng.jw_columns(100, 2000, 2)[:2]
    cases["sparse500"] = (500,) + rng.local_columns(500, 600, rng.SplitMix64(8), 500, (2, 12))[:2]
    cases["dense500"] = (500,) + cols(ref.random_sum(500, 200, 4))[:2]
    allz = np.zeros((50, 2), np.uint64)
    allz_z = r.integers(0, 2**63, size=(50, 2), dtype=np.int64).astype(np.uint64)
    allz_z[:, 1] &= np.uint64((1 << 36) - 1)
    cases["allz"] = (100, allz, allz_z)
    for name, (n, x, z) in cases.items():
        stats = ref.GroupingStats()
        part = ref.group_greedy(ref_sum(n, x, z, np.zeros(x.shape[0], np.uint8),
                                        np.ones(x.shape[0], np.complex128)), stats=stats)
        gof = np.zeros(x.shape[0], np.int32)
        for gi, g in enumerate(part.groups):
            gof[g] = gi
        save(f"group_{name}", n=np.array(n), x=x, z=z, group_of=gof,
             pair_checks=np.array(stats.pair_checks), n_groups=np.array(part.group_count()))

    # 8. bitmatrix block via the reference's own _sip_words (strings.py:47-51)
    x, z, _, _ = rng.c5_columns(700, seed=10)
    bits = ref_strings._sip_words(x[:, None, :], z[:, None, :], x[None, :, :], z[None, :, :])
    save("bitmatrix_c5", x=x, z=z, bits=bits.astype(np.uint8))
    x, z, _, _ = cols(ref.random_sum(100, 300, 13))
    bits = ref_strings._sip_words(x[:, None, :], z[:, None, :], x[None, :, :], z[None, :, :])
    save("bitmatrix_dense100", x=x, z=z, bits=bits.astype(np.uint8))


if __name__ == "__main__":
    main()
