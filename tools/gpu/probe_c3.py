import sys, time, torch, collections
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[2]))
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng, _native
dev = torch.device('cuda', 0)
x, z, f, c = rng.config_columns(3)
S = pl.PauliSumSoA.from_columns(100, x, z, f, c, device=dev)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _native.stage_timing(True)
    g, ng, pc = pl.group_assignment(S)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    _native.stage_timing(False)
    agg = collections.defaultdict(float); cnt = collections.Counter()
    for n, m in _native.stage_times():
        agg[n] += m; cnt[n] += 1
    print(it, 'wall %.1f ms' % ((t1 - t0) * 1e3), int(ng.item()), {k: (round(v, 2), cnt[k]) for k, v in agg.items()}, flush=True)
