"""Seeded instance generation (host side, numpy) for every BASELINE config.

``SplitMix64`` and ``random_sum`` restate the reference generator exactly
(``paulialg/rng.py``): a counter-based stream whose k-th draw of a call is
``mix(state + k*GOLDEN)`` (rng.py:29-44), letter code ``draw & 3`` with
0=I 1=X 2=Y 3=Z (rng.py:5-8, :56-57), coefficients uniform in [-1, 1) from the
top 53 bits (rng.py:47-49), term t consuming draws t(n+1) .. t(n+1)+n
(rng.py:73-82).  Config 1 therefore reproduces ``random_sum(500, 65536, 0/1)``
bit for bit.

Configs 2-5 are NOT defined by the reference; the generators below pin them
(see DESIGN.md "Inputs").  Every generator consumes a FIXED number of draws per
term so it vectorises; supports are drawn with Floyd's subset algorithm, bounded
integers with a 64x64 multiply-high, Gaussian coefficients with Box-Muller.
Letters and supports are integer-exact on any host.  Gaussian coefficients go
through numpy's float64 log/cos/sin, whose last-ulp results may depend on the
host CPU's SIMD dispatch; tests never compare generated coefficients across
hosts bit-exactly (inputs are generated once and fed to both oracle and GPU).
"""

from __future__ import annotations

import numpy as np

from .bits import words_for

_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_U64 = np.uint64


def _mix64(v: np.ndarray) -> np.ndarray:
    v = (v ^ (v >> _U64(30))) * _U64(0xBF58476D1CE4E5B9)
    v = (v ^ (v >> _U64(27))) * _U64(0x94D049BB133111EB)
    return v ^ (v >> _U64(31))


class SplitMix64:
    """Counter-based 64-bit stream (restates rng.py:29-44)."""

    __slots__ = ("_state",)

    def __init__(self, seed: int):
        self._state = int(seed) & _M64

    def next_array(self, count: int) -> np.ndarray:
        count = int(count)
        with np.errstate(over="ignore"):
            ctr = np.arange(1, count + 1, dtype=np.uint64) * _U64(_GOLDEN)
            out = _mix64(_U64(self._state) + ctr)
        self._state = (self._state + count * _GOLDEN) & _M64
        return out

    def next_uint64(self) -> int:
        return int(self.next_array(1)[0])


# ----------------------------------------------------------------- helpers
def _unit53(d: np.ndarray) -> np.ndarray:
    """Top 53 bits -> float64 in [0, 1)."""
    return (d >> _U64(11)).astype(np.float64) * (2.0 ** -53)


def _bounded(d: np.ndarray, bound) -> np.ndarray:
    """floor(d * bound / 2^64) for bound < 2^32: uniform-enough integer in [0, bound)."""
    bound = np.asarray(bound, dtype=np.uint64)
    hi = d >> _U64(32)
    lo = d & _U64(0xFFFFFFFF)
    with np.errstate(over="ignore"):
        return ((hi * bound) + ((lo * bound) >> _U64(32))) >> _U64(32)


def _gauss(d1: np.ndarray, d2: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Box-Muller pair of independent N(0,1) samples from two draws."""
    u1 = 1.0 - _unit53(d1)          # (0, 1]
    u2 = _unit53(d2)
    r = np.sqrt(-2.0 * np.log(u1))
    t = 2.0 * np.pi * u2
    return r * np.cos(t), r * np.sin(t)


def _floyd_subsets(draws: np.ndarray, universe: int, weight: np.ndarray) -> np.ndarray:
    """Uniform w-subsets of range(universe), one per row, via Floyd's algorithm.

    ``draws`` is (m, wmax); ``weight`` (m,) gives each row's subset size.
    Returns (m, wmax) int64 with -1 in unused slots (columns >= weight).
    """
    m, wmax = draws.shape
    out = np.full((m, wmax), -1, dtype=np.int64)
    w = weight.astype(np.int64)
    for k in range(wmax):
        active = k < w
        j = universe - w + k                       # per row: Q - w + k
        jj = np.where(active, j, 0)
        t = _bounded(draws[:, k], (jj + 1).astype(np.uint64)).astype(np.int64)
        dup = (out[:, :k] == t[:, None]).any(axis=1) if k else np.zeros(m, bool)
        pick = np.where(dup, jj, t)
        out[:, k] = np.where(active, pick, -1)
    return out


def _terms_from_support(n: int, qubits: np.ndarray, codes: np.ndarray):
    """(m, wmax) qubit indices (-1 = unused) + letter codes 1=X 2=Y 3=Z -> (x, z) (m, W)."""
    m, wmax = qubits.shape
    W = words_for(n)
    x = np.zeros((m, W), dtype=np.uint64)
    z = np.zeros((m, W), dtype=np.uint64)
    rows = np.arange(m)
    for k in range(wmax):
        q = qubits[:, k]
        ok = q >= 0
        qq = np.where(ok, q, 0)
        word = qq // 64
        bit = (np.uint64(1) << (qq % 64).astype(np.uint64))
        c = codes[:, k]
        xb = np.where(ok & ((c == 1) | (c == 2)), bit, _U64(0))
        zb = np.where(ok & (c >= 2), bit, _U64(0))
        np.bitwise_or.at(x, (rows, word), xb)
        np.bitwise_or.at(z, (rows, word), zb)
    return x, z


def _letter_codes_to_words(codes: np.ndarray, n: int):
    """(m, n) RNG letter codes (0=I 1=X 2=Y 3=Z) -> (x, z) (m, W) words (rng.py:52-63)."""
    from .bits import bits_to_words

    W = words_for(n)
    xb = ((codes == 1) | (codes == 2)).astype(np.uint8)
    zb = (codes >= 2).astype(np.uint8)
    return bits_to_words(xb, W), bits_to_words(zb, W)


# ------------------------------------------------------------ generators
def random_columns(n: int, m: int, seed: int):
    """Columns of ``random_sum(n, m, seed)`` (rng.py:73-82): x, z (m, W), flags, coeffs."""
    W = words_for(n)
    if m == 0:
        return (np.zeros((0, W), np.uint64), np.zeros((0, W), np.uint64),
                np.zeros(0, np.uint8), np.zeros(0, np.complex128))
    d = SplitMix64(seed).next_array(m * (n + 1)).reshape(m, n + 1)
    codes = (d[:, :n] & _U64(3)).astype(np.uint8)
    coeffs = ((d[:, n] >> _U64(11)).astype(np.float64) * (2.0 ** -52) - 1.0).astype(np.complex128)
    x, z = _letter_codes_to_words(codes, n)
    return x, z, np.zeros(m, np.uint8), coeffs


def random_sum(n: int, m: int, seed: int, *, layout: str = "aos"):
    """Uniform random sum, identical draws to the reference ``random_sum``
    (rng.py:73-82).  Returns the reference's packed ``PauliSum`` by default;
    ``layout="soa"`` gives device-ready ``PauliSumSoA`` planes instead."""
    from .sums import PauliSum, PauliSumSoA

    cols = random_columns(n, m, seed)
    cls = PauliSumSoA if layout == "soa" else PauliSum
    return cls.from_columns(n, *cols)


def random_string(n: int, stream: SplitMix64):
    """One uniform string, phase 0 (rng.py:66-70): consumes exactly n draws of
    ``stream`` (letter code = draw & 3, 0=I 1=X 2=Y 3=Z)."""
    from .strings import PauliString

    codes = (stream.next_array(n) & _U64(3)).astype(np.uint8)[None, :]
    x, z = _letter_codes_to_words(codes, n)
    return PauliString(n, x[0], z[0], 0, validate=False)


def local_columns(n: int, m: int, stream: SplitMix64, universe: int, weight,
                  complex_coeffs: bool = True, sigma: float = 1.0):
    """m terms, each with ``weight`` distinct qubits from range(universe) and letters
    uniform over {X, Y, Z}.  ``weight`` is an int or a (lo, hi) inclusive range.

    Draw layout per term (fixed count so it vectorises):
    [weight draw] + wmax support draws + wmax letter draws + 2 coefficient draws.
    """
    if isinstance(weight, tuple):
        lo, hi = weight
        wmax, has_w = hi, 1
    else:
        lo = hi = wmax = int(weight)
        has_w = 0
    per = has_w + 2 * wmax + 2
    d = stream.next_array(m * per).reshape(m, per)
    if has_w:
        w = lo + _bounded(d[:, 0], hi - lo + 1).astype(np.int64)
    else:
        w = np.full(m, wmax, dtype=np.int64)
    sup = _floyd_subsets(d[:, has_w:has_w + wmax], universe, w)
    codes = 1 + _bounded(d[:, has_w + wmax:has_w + 2 * wmax], 3).astype(np.int64)
    x, z = _terms_from_support(n, sup, codes)
    re, im = _gauss(d[:, per - 2], d[:, per - 1])
    if complex_coeffs:
        c = re + 1j * im
    else:
        c = (sigma * re).astype(np.complex128)
    return x, z, np.zeros(m, np.uint8), c.astype(np.complex128)


def jw_columns(n: int, m: int, seed: int):
    """Config 3: Jordan-Wigner-style terms.

    Per term 12 draws: [kind, subtype, e0..e3 (Floyd), l0..l3, g1, g2].
    kind < 0.3 -> diagonal: subtype 0 single Z, 1 ZZ on two distinct qubits;
    else excitation: subtype 0 two endpoints, 1 four; endpoints sorted and
    paired (e0,e1),(e2,e3); endpoint letters X/Y uniform; Z strictly inside
    each pair.  Coefficient real N(0, 0.1).
    """
    st = SplitMix64(seed)
    d = st.next_array(m * 12).reshape(m, 12)
    diag = _unit53(d[:, 0]) < 0.3
    sub = (d[:, 1] >> _U64(63)).astype(np.int64)
    nend = np.where(diag, 1 + sub, 2 + 2 * sub)        # qubits drawn
    sup = _floyd_subsets(d[:, 2:6], n, nend)
    srt = np.sort(np.where(sup < 0, n + 1, sup), axis=1)
    W = words_for(n)
    xb = np.zeros((m, n), dtype=np.uint8)
    zb = np.zeros((m, n), dtype=np.uint8)
    rows = np.arange(m)
    lx = (d[:, 6:10] >> _U64(63)).astype(np.uint8)      # 0 -> X, 1 -> Y
    # diagonal terms: Z on the drawn qubits
    for k in range(2):
        sel = diag & (k < nend)
        zb[rows[sel], srt[sel, k]] = 1
    # excitation terms
    exc = ~diag
    qi = np.arange(n)[None, :]
    for p in range(2):
        sel = exc & (2 * p + 1 < nend)
        a = srt[:, 2 * p]
        b = srt[:, 2 * p + 1]
        for e, col in ((a, 2 * p), (b, 2 * p + 1)):
            r = rows[sel]
            xb[r, e[sel]] = 1
            zb[r, e[sel]] = lx[sel, col]
        inside = sel[:, None] & (qi > a[:, None]) & (qi < b[:, None])
        zb |= inside.astype(np.uint8)
    from .bits import bits_to_words

    x = bits_to_words(xb, W)
    z = bits_to_words(zb, W)
    re, _ = _gauss(d[:, 10], d[:, 11])
    return x, z, np.zeros(m, np.uint8), (0.1 * re).astype(np.complex128)


def config_columns(cfg: int, scale: float = 1.0):
    """Columns for BASELINE config ``cfg`` (1..5).  ``scale`` < 1 shrinks term
    counts for parity tests (the draw layout is unchanged, so a smaller config is
    a prefix of the full one for configs 2-4)."""
    if cfg == 1:
        p = max(1, int(65536 * scale))
        return random_columns(500, p, 0), random_columns(500, p, 1)
    if cfg == 2:
        m = max(1, int(1000 * scale))
        st = SplitMix64(1)
        a = local_columns(500, 1000, st, 24, 4)
        b = local_columns(500, 1000, st, 24, 4)
        return _head(a, m), _head(b, m)
    if cfg == 3:
        m = max(1, int(100_000 * scale))
        return jw_columns(100, 100_000, 2) if m == 100_000 else _head(jw_columns(100, 100_000, 2), m)
    if cfg == 4:
        m = max(1, int(10_000 * scale))
        st = SplitMix64(3)
        a = local_columns(500, 10_000, st, 48, 8)
        b = local_columns(500, 10_000, st, 48, 8)
        return _head(a, m), _head(b, m)
    if cfg == 5:
        return c5_columns(max(1, int(1_000_000 * scale)))
    raise ValueError(f"unknown config {cfg}")


def c5_columns(m: int = 1_000_000, seed: int = 4):
    """Config 5: 90% base terms (weight 2..12 over all 500 qubits) + 10% exact
    copies (string and coefficient) of uniformly chosen base terms, then a
    uniform random permutation (argsort of one draw per term, stable)."""
    st = SplitMix64(seed)
    nbase = m - m // 10
    ndup = m - nbase
    x, z, f, c = local_columns(500, nbase, st, 500, (2, 12))
    src = _bounded(st.next_array(ndup), nbase).astype(np.int64)
    x = np.concatenate([x, x[src]])
    z = np.concatenate([z, z[src]])
    f = np.concatenate([f, f[src]])
    c = np.concatenate([c, c[src]])
    order = np.argsort(st.next_array(m), kind="stable")
    return x[order], z[order], f[order], c[order]


def _head(cols, m):
    return tuple(np.ascontiguousarray(a[:m]) for a in cols)
