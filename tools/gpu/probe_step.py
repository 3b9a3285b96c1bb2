import time, torch, sys
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[2]))
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng, _native
dev = torch.device('cuda', 0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
a, b = rng.config_columns(cfg)
A = pl.PauliSumSoA.from_columns(500, *a, device=dev)
B = pl.PauliSumSoA.from_columns(500, *b, device=dev)
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _native.stage_timing(True)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    out = pl.outer_multiply(A, B)
    e1.record()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    _native.stage_timing(False)
    st = _native.stage_times()
    ms = torch.cuda.memory_stats(); extra = (ms.get('num_device_alloc'), ms.get('num_device_free'), ms.get('num_alloc_retries'))
    print(it, extra, 'wall %.1f ms  event %.1f ms' % ((t1 - t0) * 1e3, e0.elapsed_time(e1)), [(n, round(m, 2)) for n, m in st], flush=True)
    del out
