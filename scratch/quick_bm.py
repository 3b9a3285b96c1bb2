import sys, time; sys.path.insert(0, '.')
import torch
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng, _native
dev = torch.device('cuda')
x, z, f, c = rng.c5_columns(1_000_000, seed=4)
S = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=dev)
M = len(S); rows = 65536; nw = (M + 31) // 32
buf = torch.empty((rows, nw), dtype=torch.int32, device=dev)
def run():
    for r0 in range(0, M, rows):
        r = min(rows, M - r0)
        pl.commutation_bitmatrix(S, row0=r0, rows=r, out=buf[:r])
run(); torch.cuda.synchronize()
_native.stage_timing(True)
t0 = time.perf_counter(); run(); torch.cuda.synchronize(); t1 = time.perf_counter()
_native.stage_timing(False)
st = _native.stage_times()
k = sum(ms for n, ms in st if n.startswith('k_bitmatrix'))
print(f"bitmatrix full: {1e3*(t1-t0):.1f} ms wall, kernels {k:.1f} ms, {M*M/(t1-t0):.3e} checks/s, out {M*nw*4/(t1-t0)/1e9:.0f} GB/s")
