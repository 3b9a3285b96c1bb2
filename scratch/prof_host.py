import sys, time; sys.path.insert(0, '.')
import torch, ctypes as C
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng, _native, sums
from paper_2605_25974_b200._device import ptr, stream_ptr
dev = torch.device('cuda')
a, b = rng.config_columns(4)
A = pl.PauliSumSoA.from_columns(500, *a, device=dev); B = pl.PauliSumSoA.from_columns(500, *b, device=dev)
for _ in range(3): out = pl.outer_multiply(A, B); del out
torch.cuda.synchronize()
def T(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(3):
    t0 = T()
    Ap = A.planes(); Bp = B.planes(); st = stream_ptr(dev)
    plan = _native.MergePlan()
    _native.call("pl_outer_plan", 8, len(A), len(B), ptr(Ap.x), ptr(Ap.z), Ap.ld, ptr(Bp.x), ptr(Bp.z), Bp.ld, C.byref(plan), st)
    t1 = T()
    ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev)
    x, z, k, c = sums._alloc_planes(8, plan.n_items, dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    t2 = T()
    _native.call("pl_outer_multiply_combine", C.byref(plan), ptr(Ap.x), ptr(Ap.z), ptr(Ap.k), ptr(Ap.c), Ap.ld,
                 ptr(Bp.x), ptr(Bp.z), ptr(Bp.k), ptr(Bp.c), Bp.ld, 0.0, ptr(ws), ws.numel(),
                 ptr(x), ptr(z), ptr(k), ptr(c), x.stride(0), ptr(cnt), st)
    t3h = time.perf_counter()
    t3 = T()
    m = int(cnt.item())
    t4 = T()
    print(f"plan {1e3*(t1-t0):.2f} alloc {1e3*(t2-t1):.2f} launch(host) {1e3*(t3h-t2):.2f} gpu {1e3*(t3-t2):.2f} count {1e3*(t4-t3):.2f} ms")
    del ws, x, z, k, c
_native.stage_timing(True)
out = pl.outer_multiply(A, B); torch.cuda.synchronize()
print(_native.stage_times())
