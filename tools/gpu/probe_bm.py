import sys, torch, time
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[2]))
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng, _native
dev = torch.device('cuda', 0)
x, z, f, c = rng.c5_columns(1_000_000, seed=4)
S = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=dev)
M = len(S)
rows = 65536
nw = (M + 31) // 32
buf = torch.empty((rows, nw), dtype=torch.int32, device=dev)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for it in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _native.stage_timing(True)
    pl.commutation_bitmatrix(S, row0=0, rows=rows, out=buf)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    _native.stage_timing(False)
    print(it, '%.2f ms' % ((t1 - t0) * 1e3), [(n, round(m, 3)) for n, m in _native.stage_times()], flush=True)
