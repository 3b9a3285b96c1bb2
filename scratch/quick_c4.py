import sys, time; sys.path.insert(0, '.')
import torch
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng, _native
dev = torch.device('cuda')
for cfg, scale in ((4, 1.0), (2, 1.0)):
    a, b = rng.config_columns(cfg, scale)
    A = pl.PauliSumSoA.from_columns(500, *a, device=dev); B = pl.PauliSumSoA.from_columns(500, *b, device=dev)
    for _ in range(3): out = pl.outer_multiply(A, B); del out
    torch.cuda.synchronize()
    _native.stage_timing(True)
    t0 = time.perf_counter()
    for _ in range(3): out = pl.outer_multiply(A, B); del out
    torch.cuda.synchronize(); t1 = time.perf_counter()
    _native.stage_timing(False)
    agg = {}
    for n, ms in _native.stage_times(): agg[n] = agg.get(n, 0) + ms / 3
    print(f"C{cfg}: {1e3*(t1-t0)/3:.2f} ms/step", {k: round(v, 3) for k, v in agg.items()})
