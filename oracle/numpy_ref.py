"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference hot path.

Term-major (M, W) uint64 "columns", exactly as the reference's kernels see
them (sums.py:240-242).  Each function cites the reference code it restates.
"""

from __future__ import annotations

import numpy as np

_PHASE = np.array([1.0, 1.0j, -1.0, -1.0j], dtype=np.complex128)  # bits.py:19


def _pc(a: np.ndarray) -> np.ndarray:
    """Row sums of per-word popcounts (bits.py:49-51 + the .sum(axis=-1) idiom)."""
    return np.bitwise_count(a).sum(axis=-1, dtype=np.int64)


def phase_exponent(ax, az, bx, bz) -> np.ndarray:
    """k of the letter product a*b mod 4 (strings.py:32-44)."""
    k = _pc(ax & az) + _pc(bx & bz) + 2 * _pc(az & bx) - _pc((ax ^ bx) & (az ^ bz))
    return np.mod(k, 4)


def sip(ax, az, bx, bz) -> np.ndarray:
    """Symplectic product parity, 1 = anti-commute (strings.py:47-51)."""
    return (_pc(ax & bz) + _pc(az & bx)) & 1


def batch_pair_multiply(ax, az, aflags, bx, bz, bflags):
    """bench.py:168-177: elementwise products of aligned term arrays."""
    k = aflags.astype(np.int64) + bflags.astype(np.int64) + phase_exponent(ax, az, bx, bz)
    return ax ^ bx, az ^ bz, np.mod(k, 4).astype(np.uint8)


def outer_raw(ax, az, af, ac, bx, bz, bf, bc, threads: int = 1, chunk: int = 1 << 16):
    """sums.py:123-174: row j*Ma + i = a_i * b_j (j-major), coeff a_c[i]*b_c[j].

    ``threads`` splits the j range over a thread pool like sums.py:158-173;
    outputs are disjoint per block, so the result is thread-count independent.
    """
    ma, W = ax.shape
    mb = bx.shape[0]
    out_x = np.empty((ma * mb, W), np.uint64)
    out_z = np.empty((ma * mb, W), np.uint64)
    out_k = np.empty(ma * mb, np.uint8)
    out_c = np.empty(ma * mb, np.complex128)
    ka = af.astype(np.int64) + _pc(ax & az)          # sums.py:156
    kb = bf.astype(np.int64) + _pc(bx & bz)          # sums.py:157

    def block(j0: int, j1: int) -> None:
        step = max(1, chunk // max(ma, 1))           # sums.py:127
        for js in range(j0, j1, step):
            je = min(j1, js + step)
            bxs, bzs = bx[js:je, None, :], bz[js:je, None, :]
            x = ax[None] ^ bxs
            z = az[None] ^ bzs
            k = ka[None, :] + kb[js:je, None] + 2 * _pc(az[None] & bxs) - _pc(x & z)
            rows = slice(js * ma, je * ma)
            out_x[rows] = x.reshape(-1, W)
            out_z[rows] = z.reshape(-1, W)
            out_k[rows] = np.mod(k, 4).reshape(-1)
            out_c[rows] = (ac[None, :] * bc[js:je, None]).reshape(-1)

    if threads <= 1 or mb < 2:
        block(0, mb)
    else:
        from concurrent.futures import ThreadPoolExecutor

        cuts = np.linspace(0, mb, threads + 1).astype(int)
        with ThreadPoolExecutor(threads) as pool:
            list(pool.map(lambda t: block(int(cuts[t]), int(cuts[t + 1])), range(threads)))
    return out_x, out_z, out_k, out_c


def outer_raw_rows(ax, az, af, ac, bx, bz, bf, bc, rows):
    """Selected rows r = j*Ma + i of the raw outer product (sums.py:123-141):
    x = a_x ^ b_x, z = a_z ^ b_z, k = (base_a + base_b + 2popc(az&bx) -
    popc(x&z)) mod 4 with base = flags + popc(x&z) (sums.py:156-157), coeff
    a_c[i]*b_c[j].  Rows come out in the given order."""
    ma = ax.shape[0]
    rows = np.asarray(rows, dtype=np.int64)
    j, i = np.divmod(rows, ma)
    axs, azs, bxs, bzs = ax[i], az[i], bx[j], bz[j]
    x, z = axs ^ bxs, azs ^ bzs
    k = (af[i].astype(np.int64) + _pc(axs & azs) + bf[j].astype(np.int64) + _pc(bxs & bzs)
         + 2 * _pc(azs & bxs) - _pc(x & z))
    return x, z, np.mod(k, 4).astype(np.uint8), ac[i] * bc[j]


def canonical_order(x, z) -> np.ndarray:
    """Stable permutation sorting rows by (z_0..z_{W-1}, x_0..x_{W-1}) as unsigned
    words, z_0 most significant (sums.py:104-106, strings.py:165-167)."""
    W = x.shape[1]
    keys = np.concatenate([z, x], axis=1)            # columns in priority order
    return np.lexsort(tuple(keys[:, c] for c in range(2 * W - 1, -1, -1)))


def combine(x, z, flags, coeffs, eps: float = 0.0):
    """sums.py:94-120: fold i^k, sort, merge equal keys, drop |c| <= eps, flags 0."""
    m = x.shape[0]
    c = coeffs * _PHASE[flags]
    if m == 0:
        return x.copy(), z.copy(), flags.copy(), c
    order = canonical_order(x, z)
    xs, zs, cs = x[order], z[order], c[order]
    new_run = np.ones(m, dtype=bool)
    new_run[1:] = (xs[1:] != xs[:-1]).any(axis=1) | (zs[1:] != zs[:-1]).any(axis=1)
    heads = np.flatnonzero(new_run)
    sums = np.add.reduceat(cs, heads)
    keep = np.abs(sums) > eps
    heads = heads[keep]
    return (np.ascontiguousarray(xs[heads]), np.ascontiguousarray(zs[heads]),
            np.zeros(heads.size, np.uint8), sums[keep])


def outer_combine(ax, az, af, ac, bx, bz, bf, bc, eps: float = 0.0, threads: int = 1):
    """sums.py:293-305 with combine=True."""
    return combine(*outer_raw(ax, az, af, ac, bx, bz, bf, bc, threads=threads), eps)


def greedy(x, z):
    """grouping.py:67-95: first-fit over groups in creation order.

    Returns (groups, pair_checks) where pair_checks counts, like
    grouping.py:75-76, the members of every group tried.
    """
    groups: list[list[int]] = []
    gx: list[np.ndarray] = []
    gz: list[np.ndarray] = []
    checks = 0
    for t in range(x.shape[0]):
        xt, zt = x[t], z[t]
        for gi, g in enumerate(groups):
            checks += len(g)
            if not sip(xt, zt, gx[gi], gz[gi]).any():
                g.append(t)
                gx[gi] = np.vstack([gx[gi], xt[None]])
                gz[gi] = np.vstack([gz[gi], zt[None]])
                break
        else:
            groups.append([t])
            gx.append(xt[None].copy())
            gz.append(zt[None].copy())
    return groups, checks


def pair_checks_from_assignment(group_of: np.ndarray) -> int:
    """Recompute grouping.py:75-76's counter from a final assignment: term t
    tried every group up to and including its own, whose sizes at time t count
    the earlier terms u < t with group(u) <= group(t)."""
    g = np.asarray(group_of, dtype=np.int64)
    m = g.size
    if m == 0:
        return 0
    ng = int(g.max()) + 1
    tree = np.zeros(ng + 1, dtype=np.int64)          # Fenwick over group ids
    total = 0
    for t in range(m):
        i = int(g[t]) + 1
        s = 0
        while i > 0:
            s += int(tree[i])
            i -= i & -i
        total += s
        i = int(g[t]) + 1
        while i <= ng:
            tree[i] += 1
            i += i & -i
    return total


def bitmatrix(x, z, r0: int, r1: int, c0: int, c1: int) -> np.ndarray:
    """(r1-r0, c1-c0) uint8 anti-commutation matrix: the all-pairs block of
    grouping.py:136-140 (popc(x_r & z_c) + popc(z_r & x_c)) & 1."""
    xr, zr = x[r0:r1, None, :], z[r0:r1, None, :]
    xc, zc = x[None, c0:c1, :], z[None, c0:c1, :]
    return ((_pc(xr & zc) + _pc(zr & xc)) & 1).astype(np.uint8)


def pack_bitrows(bits: np.ndarray) -> np.ndarray:
    """(R, C) 0/1 -> (R, ceil(C/32)) uint32, bit c%32 of word c//32."""
    r, c = bits.shape
    nw = (c + 31) // 32
    pad = np.zeros((r, nw * 32), np.uint8)
    pad[:, :c] = bits
    return np.packbits(pad, axis=1, bitorder="little").view("<u4").astype(np.uint32).reshape(r, nw)


# ---------------------------------------------------------------- §8(f) f1/f2
def apply_clifford(x, z, flags, gate: str, qubits, n: int):
    """U P U^dagger over every row (gates.py:31-102), returned as copies.
    H: swap the x/z bits, sign flip where the letter is Y; S: z ^= x, flip
    where Y; CNOT(c,t): x_t ^= x_c, z_c ^= z_t, flip where x_c z_t (x_t ^ z_c ^ 1);
    CZ(c,t): z_c ^= x_t, z_t ^= x_c, flip where x_c x_t (z_c ^ z_t)."""
    x, z, f = x.copy(), z.copy(), flags.copy()
    one = np.uint64(1)

    def bit(a, q):
        return (a[:, q // 64] >> np.uint64(q % 64)) & one

    gate = gate.upper()
    if gate in ("H", "S"):
        (q,) = qubits
        w, m = q // 64, np.uint64(1 << (q % 64))
        xb, zb = x[:, w] & m, z[:, w] & m
        if gate == "H":
            f ^= (((xb & zb) != 0).astype(np.uint8) << 1)
            x[:, w] = (x[:, w] & ~m) | zb
            z[:, w] = (z[:, w] & ~m) | xb
        else:
            f ^= (((xb & z[:, w]) != 0).astype(np.uint8) << 1)
            z[:, w] ^= xb
        return x, z, f
    c, t = qubits
    xc, zc, xt, zt = bit(x, c), bit(z, c), bit(x, t), bit(z, t)
    if gate == "CNOT":
        cond = xc & zt & (xt ^ zc ^ one)
        x[:, t // 64] ^= xc << np.uint64(t % 64)
        z[:, c // 64] ^= zt << np.uint64(c % 64)
    else:
        cond = xc & xt & (zc ^ zt)
        z[:, c // 64] ^= xt << np.uint64(c % 64)
        z[:, t // 64] ^= xc << np.uint64(t % 64)
    f ^= (cond.astype(np.uint8) << 1)
    return x, z, f


def rotation_split(x, z, flags, coeffs, gx, gz, cos_t: float, sin_t: float):
    """Un-combined rotation split (sums.py:177-223): commuting rows pass,
    an anti-commuting row becomes (c*cos, Q) then (c*(-1j*sin)*i^k, P*Q
    letters, flags 0), k = flags + phase(P, Q); sin == 0 scales, cos == 0
    replaces in place."""
    gxm = np.broadcast_to(gx, x.shape)
    gzm = np.broadcast_to(gz, z.shape)
    anti = sip(x, z, gxm, gzm).astype(bool)
    m, words = x.shape
    if sin_t == 0.0:
        return x.copy(), z.copy(), flags.copy(), np.where(anti, coeffs * cos_t, coeffs)
    pk = (flags[anti].astype(np.int64) + phase_exponent(gxm[anti], gzm[anti], x[anti], z[anti])) % 4
    prod = coeffs[anti] * (-1j * sin_t) * _PHASE[pk]
    if cos_t == 0.0:
        ox, oz, of, oc = x.copy(), z.copy(), flags.copy(), coeffs.copy()
        ox[anti] ^= gx
        oz[anti] ^= gz
        of[anti] = 0
        oc[anti] = prod
        return ox, oz, of, oc
    total = m + int(anti.sum())
    first = np.cumsum(np.concatenate(([0], 1 + anti.astype(np.int64))))[:m]
    second = first[anti] + 1
    ox = np.empty((total, words), np.uint64)
    oz = np.empty((total, words), np.uint64)
    of = np.empty(total, np.uint8)
    oc = np.empty(total, np.complex128)
    ox[first], oz[first], of[first] = x, z, flags
    oc[first] = np.where(anti, coeffs * cos_t, coeffs)
    ox[second], oz[second], of[second], oc[second] = x[anti] ^ gx, z[anti] ^ gz, 0, prod
    return ox, oz, of, oc


def greedy_parallel(x, z, chunks: int):
    """Two-phase grouping (grouping.py:98-146): greedy per contiguous chunk
    (np.array_split), then each local group joins the first global group all
    of whose cross pairs commute, else opens one.  Returns (groups in member
    order, pair_checks)."""
    m = x.shape[0]
    pieces = [p for p in np.array_split(np.arange(m), chunks) if p.size]
    checks = 0
    locals_ = []
    for p in pieces:
        groups_l, c = greedy(x[p], z[p])
        checks += int(c)
        locals_.extend([[int(p[0]) + t for t in g] for g in groups_l])
    glob: list[list[int]] = []
    for loc in locals_:
        lx, lz = x[loc], z[loc]
        placed = False
        for g in glob:
            checks += len(loc) * len(g)
            gx, gz = x[g], z[g]
            cross = _pc(lx[:, None, :] & gz[None, :, :]) + _pc(lz[:, None, :] & gx[None, :, :])
            if not (cross & 1).any():
                g.extend(loc)
                placed = True
                break
        if not placed:
            glob.append(list(loc))
    return glob, checks
