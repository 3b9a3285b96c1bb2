"""Latency of the scalar string API (PauliString.multiply / commutes)."""
import sys, time
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[2]))
import numpy as np
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng
s = rng.SplitMix64(5)
a = [pl.random_string(500, s) for _ in range(64)]
b = [pl.random_string(500, s) for _ in range(64)]
for _ in range(2):
    t0 = time.perf_counter()
    for p, q in zip(a, b):
        r = p.multiply(q)
    t1 = time.perf_counter()
    for p, q in zip(a, b):
        c = p.commutes(q)
    t2 = time.perf_counter()
    print('multiply %.1f us/op  commutes %.1f us/op' % ((t1 - t0) / 64 * 1e6, (t2 - t1) / 64 * 1e6), flush=True)
