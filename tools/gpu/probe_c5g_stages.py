"""Stage times of the full C5 grouping (10^6 terms, n=500)."""
import sys, time, torch, collections
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[2]))
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng, _native
dev = torch.device('cuda', 0)
x, z, f, c = rng.c5_columns(1_000_000)
S = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=dev)
pl.group_assignment(S)
for it in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if it: _native.stage_timing(True)
    g, ng, pc = pl.group_assignment(S)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    _native.stage_timing(False)
    agg = collections.defaultdict(float); cnt = collections.Counter()
    for n, m in (_native.stage_times(16384) if it else []):
        agg[n] += m; cnt[n] += 1
    print(it, 'wall %.1f ms' % ((t1 - t0) * 1e3), int(ng.item()), {k: (round(v, 2), cnt[k]) for k, v in agg.items()}, flush=True)
