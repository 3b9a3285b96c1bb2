import sys, time; sys.path.insert(0, '.')
import torch, numpy as np
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng, _native
dev = torch.device('cuda')
x, z, f, c = rng.config_columns(3)
S = pl.PauliSumSoA.from_columns(100, x, z, f, c, device=dev)
for name, s in (("C3", S),):
    pl.group_assignment(s); torch.cuda.synchronize()
    _native.stage_timing(True)
    t0 = time.perf_counter(); gof, ng, pc = pl.group_assignment(s); torch.cuda.synchronize(); t1 = time.perf_counter()
    _native.stage_timing(False)
    agg = {}
    for n, ms in _native.stage_times(): agg[n] = agg.get(n, 0) + ms
    print(name, f"{1e3*(t1-t0):.1f} ms groups {int(ng)} checks {int(pc)} -> {int(pc)/(t1-t0):.3e} checks/s", {k: round(v, 2) for k, v in agg.items()})
x, z, f, c = rng.c5_columns(1_000_000, seed=4)
for m in (100_000, 1_000_000):
    s = pl.PauliSumSoA.from_columns(500, x[:m], z[:m], f[:m], c[:m], device=dev)
    _native.stage_timing(True)
    t0 = time.perf_counter(); gof, ng, pc = pl.group_assignment(s); torch.cuda.synchronize(); t1 = time.perf_counter()
    _native.stage_timing(False)
    agg = {}
    for n, ms in _native.stage_times(): agg[n] = agg.get(n, 0) + ms
    print(f"C5[:{m}]", f"{1e3*(t1-t0):.1f} ms groups {int(ng)} checks {int(pc)} -> {int(pc)/(t1-t0):.3e} checks/s", {k: round(v, 2) for k, v in agg.items()})
