"""Host clear of pinned memory: torch zero_() vs glibc memset from 16 threads
(large memsets use non-temporal stores: no read-for-ownership)."""
import ctypes, time, torch
from concurrent.futures import ThreadPoolExecutor
n = 1 << 29
h = torch.empty(n, dtype=torch.int64, pin_memory=True)
d = torch.zeros(n, dtype=torch.int64, device='cuda')
libc = ctypes.CDLL(None)
libc.memset.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t]
libc.memset.restype = ctypes.c_void_p
def clear(nthreads):
    base, nbytes = h.data_ptr(), n * 8
    step = (nbytes // nthreads + 4095) & ~4095
    def one(i):
        lo = i * step
        if lo < nbytes: libc.memset(base + lo, 0, min(step, nbytes - lo))
    with ThreadPoolExecutor(nthreads) as ex: list(ex.map(one, range(nthreads)))
for nt in (8, 16, 32):
    for _ in range(2):
        t0 = time.perf_counter(); clear(nt); t1 = time.perf_counter()
    print('memset x%d %.1f GB/s' % (nt, n * 8 / (t1 - t0) / 1e9))
for _ in range(2):
    t0 = time.perf_counter(); h.zero_(); t1 = time.perf_counter()
print('torch zero_ %.1f GB/s' % (n * 8 / (t1 - t0) / 1e9))
pool = ThreadPoolExecutor(16)
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h[: n // 2].copy_(d[: n // 2], non_blocking=True)
    base, nbytes = h.data_ptr() + n * 4, n * 4
    step = (nbytes // 16 + 4095) & ~4095
    list(pool.map(lambda i: libc.memset(base + i * step, 0, max(0, min(step, nbytes - i * step))), range(16)))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print('half copy + half memset x16: %.1f GB/s effective' % (n * 8 / (t1 - t0) / 1e9))
