import time, torch, sys
sys.path.insert(0, '.')
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng, _native
from torch.profiler import profile, ProfilerActivity
dev = torch.device('cuda', 0)
a, b = rng.config_columns(4)
A = pl.PauliSumSoA.from_columns(500, *a, device=dev)
B = pl.PauliSumSoA.from_columns(500, *b, device=dev)
for it in range(3):
    out = pl.outer_multiply(A, B); del out
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for it in range(8):
        t0 = time.perf_counter()
        out = pl.outer_multiply(A, B)
        torch.cuda.synchronize()
        print(it, '%.1f ms' % ((time.perf_counter() - t0) * 1e3), flush=True)
        del out
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
prof.export_chrome_trace("gpurun_out/trace.json")
