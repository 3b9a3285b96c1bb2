import sys, time, torch
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[2]))
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng, _native
dev = torch.device('cuda', 0)
x, z, f, c = rng.config_columns(3)
S = pl.PauliSumSoA.from_columns(100, x, z, f, c, device=dev)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _native.stage_timing(True)
    st = pl.GroupingStats()
    p = pl.group_greedy_parallel(S, 8, stats=st)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    _native.stage_timing(False)
    ts = _native.stage_times()
    agg = {}
    for n, m in ts: agg[n] = agg.get(n, 0) + m
    print(it, 'wall %.1f ms' % ((t1 - t0) * 1e3), p.group_count(), st.pair_checks, {k: round(v, 2) for k, v in agg.items()}, flush=True)
