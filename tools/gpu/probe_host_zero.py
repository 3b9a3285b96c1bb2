"""Host-side zero fill bandwidth of pinned memory vs the D2H copy rate (decides
whether provably-zero output planes are cheaper to clear on the host than to copy)."""
import time, torch
n = 1 << 29  # 4 GiB of int64
h = torch.empty(n, dtype=torch.int64, pin_memory=True)
d = torch.zeros(n, dtype=torch.int64, device='cuda')
print('threads', torch.get_num_threads())
for it in range(3):
    t0 = time.perf_counter(); h.zero_(); t1 = time.perf_counter()
    print('zero_ %.1f GB/s' % (n * 8 / (t1 - t0) / 1e9))
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    print('d2h %.1f GB/s' % (n * 8 / (t1 - t0) / 1e9))
# both at once: copy half while zeroing the other half
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h[: n // 2].copy_(d[: n // 2], non_blocking=True); h[n // 2:].zero_(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print('half copy + half zero: %.1f GB/s effective' % (n * 8 / (t1 - t0) / 1e9))
