import time, torch, sys
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[2]))
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng, _native
dev = torch.device('cuda', 0)
x, z, f, c = rng.config_columns(5)
S = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=dev)
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _native.stage_timing(True)
    out = pl.sort_combine(S)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    _native.stage_timing(False)
    st = _native.stage_times()
    print(it, len(out), 'wall %.2f ms' % ((t1 - t0) * 1e3), [(n, round(m, 3)) for n, m in st], pl.sums.LAST_PLAN, flush=True)
