"""Round-2 golden fixtures, made by RUNNING THE REFERENCE (paulialg) in the
build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_r2.py

* ``rng_string``      -- rng.random_string (rng.py:66-70): consecutive strings
                         of one SplitMix64 stream, plus the stream's next draw
* ``string_clifford`` -- PauliString.apply_clifford (strings.py:153-163) on
                         single strings with phases, every gate
* ``neg_eps``         -- sum_multiply(H, H, eps=-1) and apply_rotation(eps=-1):
                         a negative eps keeps exact zeros (sums.py:113-114)
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
from paulialg.sums import PauliSum as RefSum  # noqa: E402

from paper_2605_25974_b200 import rng  # noqa: E402


def cols(s):
    x, z, f, c = s._columns()
    return (np.ascontiguousarray(x), np.ascontiguousarray(z), np.asarray(f).copy(),
            np.asarray(c).copy())


def save(name, **arrs):
    np.savez_compressed(HERE / f"{name}.npz", **arrs)
    print(name, {k: v.shape for k, v in arrs.items()})


def main():
    # random_string: 3 strings from one stream per (n, seed), then the next draw
    out = {}
    for n, seed in ((5, 0), (100, 7), (500, 3)):
        st = ref.SplitMix64(seed)
        xs, zs = [], []
        for _ in range(3):
            p = ref.random_string(n, st)
            xs.append(p.x.copy())
            zs.append(p.z.copy())
        out[f"x_{n}_{seed}"] = np.stack(xs)
        out[f"z_{n}_{seed}"] = np.stack(zs)
        out[f"next_{n}_{seed}"] = np.array(st.next_uint64(), dtype=np.uint64)
    save("rng_string", **out)

    # single-string Clifford conjugation with phases
    r = np.random.default_rng(77)
    gates = [("H", (3,)), ("S", (0,)), ("CNOT", (1, 70)), ("CZ", (65, 2)), ("H", (99,)),
             ("S", 64), ("CNOT", (99, 0)), ("CZ", (10, 11))]
    st = ref.SplitMix64(11)
    xs, zs, ks, ox, oz, ok = [], [], [], [], [], []
    for t in range(40):
        p = ref.random_string(100, st)
        k = int(r.integers(0, 4))
        p = ref.PauliString(100, p.x, p.z, k)
        g, q = gates[t % len(gates)]
        o = p.apply_clifford(g, q)
        xs.append(p.x.copy()); zs.append(p.z.copy()); ks.append(k)
        ox.append(o.x.copy()); oz.append(o.z.copy()); ok.append(o.phase)
    save("string_clifford", x=np.stack(xs), z=np.stack(zs), k=np.array(ks, np.uint8),
         ox=np.stack(ox), oz=np.stack(oz), ok=np.array(ok, np.uint8))

    # negative eps: H*H keeps the cancelled terms as exact zeros
    h = rng.local_columns(64, 60, rng.SplitMix64(5), 10, 3)
    H = RefSum._from_columns(64, *h)
    hh = ref.sum_multiply(H, H, eps=-1.0)
    hx, hz, hf, hc = cols(hh)
    gen = ref.PauliString.from_label("XZ" + "I" * 62)
    rot = ref.RotationSpec(gen, np.pi)  # cos = -1, sin = 0: exact, no split
    rr = H.apply_rotation(rot, eps=-1.0)
    rx, rz, rf, rc = cols(rr)
    save("neg_eps", hx=h[0], hz=h[1], hf=h[2], hc=h[3], ox=hx, oz=hz, ok=hf, oc=hc,
         rot_label=np.array("XZ" + "I" * 62), rx=rx, rz=rz, rf=rf, rc=rc)


if __name__ == "__main__":
    main()
