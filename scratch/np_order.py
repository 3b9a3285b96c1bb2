import numpy as np
def pw(t):
    L = len(t)
    if L < 4:
        r = complex(-0.0, -0.0)
        rr, ri = -0.0, -0.0
        for e in t:
            rr += e.real; ri += e.imag
        return rr, ri
    if L <= 64:
        R = [t[0].real, t[0].imag, t[1].real, t[1].imag, t[2].real, t[2].imag, t[3].real, t[3].imag]
        i = 4
        while i < L - (L % 4):
            R[0] += t[i].real; R[1] += t[i].imag
            R[2] += t[i+1].real; R[3] += t[i+1].imag
            R[4] += t[i+2].real; R[5] += t[i+2].imag
            R[6] += t[i+3].real; R[7] += t[i+3].imag
            i += 4
        rr = (R[0] + R[2]) + (R[4] + R[6]); ri = (R[1] + R[3]) + (R[5] + R[7])
        while i < L:
            rr += t[i].real; ri += t[i].imag; i += 1
        return rr, ri
    n2 = L  # floats in first half = n/2 where n = 2L floats
    n2 -= n2 % 8
    e1 = n2 // 2
    a = pw(t[:e1]); b = pw(t[e1:])
    return a[0] + b[0], a[1] + b[1]
def red(seg):
    if len(seg) == 1: return seg[0]
    rr, ri = pw(seg[1:])
    return complex(seg[0].real + rr, seg[0].imag + ri)
r = np.random.default_rng(1)
bad = 0; tot = 0
for L in list(range(1, 80)) + [100, 127, 128, 129, 200, 300, 513, 1000, 4097]:
    for trial in range(20):
        seg = (r.normal(size=L) * 10.0 ** r.integers(-8, 8, L)) + 1j * (r.normal(size=L) * 10.0 ** r.integers(-8, 8, L))
        got = np.add.reduceat(seg, [0])[0]
        mine = red(list(seg))
        tot += 1
        if got != mine:
            bad += 1
            if bad < 5: print("mismatch L", L, got, mine)
print("bad", bad, "of", tot)
# reduceat with multiple segments
seg = r.normal(size=50) + 1j*r.normal(size=50)
idx = np.array([0, 3, 10, 11, 40])
got = np.add.reduceat(seg, idx)
mine = [red(list(seg[a:b])) for a, b in zip(idx, list(idx[1:]) + [50])]
print("multi", all(g == m for g, m in zip(got, mine)))
