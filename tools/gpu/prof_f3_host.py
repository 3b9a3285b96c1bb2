import sys, time, torch, cProfile, pstats
sys.path.insert(0, '.')
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng
dev = torch.device('cuda', 0)
x, z, f, c = rng.config_columns(3)
S = pl.PauliSumSoA.from_columns(100, x, z, f, c, device=dev)
for _ in range(2): pl.group_greedy_parallel(S, 8)
t0=time.perf_counter(); p = pl.group_greedy_parallel(S, 8); torch.cuda.synchronize(); print('f3 wall %.1f ms' % ((time.perf_counter()-t0)*1e3))
t0=time.perf_counter(); p = pl.group_greedy(S); torch.cuda.synchronize(); print('group_greedy wall %.1f ms' % ((time.perf_counter()-t0)*1e3))
pr = cProfile.Profile(); pr.enable(); pl.group_greedy_parallel(S, 8); pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(14)
