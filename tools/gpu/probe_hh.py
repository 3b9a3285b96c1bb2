"""Repeated-key cliff: H*H for growing |H| (the identity run has length |H|)."""
import sys
import time

import torch

sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))
import paper_2605_25974_b200 as pl  # noqa: E402
from paper_2605_25974_b200 import rng, _native  # noqa: E402

dev = torch.device("cuda", 0)
for m in (1000, 4000, 10000):
    h = rng.local_columns(500, m, rng.SplitMix64(7), 48, 8)
    H = pl.PauliSumSoA.from_columns(500, *h, device=dev)
    for it in range(2):
        torch.cuda.synchronize()
        _native.stage_timing(True)
        t0 = time.perf_counter()
        out = H * H
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        _native.stage_timing(False)
        st = [(n, round(v, 3)) for n, v in _native.stage_times() if v > 0.05]
        print(f"|H|={m} it={it} {dt * 1e3:.2f} ms terms={len(out)}", st, flush=True)
