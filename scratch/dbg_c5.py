import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch, ctypes as C
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng, _native
from paper_2605_25974_b200._device import ptr, stream_ptr
from oracle import numpy_ref as R
dev = torch.device('cuda')
x, z, f, c = rng.c5_columns(5000, seed=1)
cols = (np.concatenate([x, x]), np.concatenate([z, z]), np.concatenate([f, f]), np.concatenate([c, -c]))
s = pl.PauliSumSoA.from_columns(500, *cols, device=dev)
S = s.planes()
plan = _native.MergePlan()
_native.call("pl_sort_plan", S.W, S.M, ptr(S.x), ptr(S.z), S.ld, C.byref(plan), stream_ptr(dev))
print("KW", plan.key_words, "bits", plan.key_bits, "nb", plan.n_buckets, "ns", plan.n_samples, "cap", plan.leaf_cap, "tgt", plan.leaf_target, "maxsub", plan.max_sub, "ws", plan.workspace_bytes)
ws = torch.zeros(plan.workspace_bytes, dtype=torch.uint8, device=dev)
W, m = S.W, S.M
ox = torch.empty((W, m), dtype=torch.int64, device=dev); oz = torch.empty_like(ox)
ok = torch.empty(m, dtype=torch.uint8, device=dev); oc = torch.empty(m, dtype=torch.complex128, device=dev)
cnt = torch.zeros(1, dtype=torch.int64, device=dev)
_native.call("pl_sort_combine", C.byref(plan), ptr(S.x), ptr(S.z), ptr(S.k), ptr(S.c), S.ld, 0.0, ptr(ws), ws.numel(), ptr(ox), ptr(oz), ptr(ok), ptr(oc), m, ptr(cnt), stream_ptr(dev))
torch.cuda.synchronize()
print("count", int(cnt))
KW, nb, n = plan.key_words, plan.n_buckets, m
al = lambda v: (v + 255) & ~255
o = 0
def take(nbytes):
    global o
    a = o; o = al(o + nbytes); return a
off_split = take(8*KW*nb); off_bcount = take(4*nb); off_bbase = take(4*(nb+1)); off_bcur = take(4*nb)
off_loff = take(4*(nb+1)); off_nl = take(4); off_lc = take(4); maxl = nb*plan.max_sub
off_stat = take(8*maxl); off_desc = take(16*maxl); off_k1 = take(8*KW*n); off_i1 = take(4*n); off_k2 = take(8*KW*n); off_i2 = take(4*n)
wsh = ws.cpu().numpy()
u32 = lambda a, k: wsh[a:a+4*k].view(np.uint32)
u64 = lambda a, k: wsh[a:a+8*k].view(np.uint64)
bcount = u32(off_bcount, nb); bbase = u32(off_bbase, nb+1); loff = u32(off_loff, nb+1); nl = u32(off_nl, 1)[0]
print("sum bcount", bcount.sum(), "max", bcount.max(), "n_leaves", nl, "leafctr", u32(off_lc,1)[0])
print("bcount", bcount.tolist())
desc = u32(off_desc, 4*maxl).reshape(-1, 4)[:nl]
print("desc sizes sum", desc[:, 2].sum(), "bufs", np.bincount(desc[:, 0]))
split = u64(off_split, KW*nb).reshape(KW, nb)[:, :nb-1]
k1 = u64(off_k1, KW*n).reshape(KW, n); i1 = u32(off_i1, n)
k2 = u64(off_k2, KW*n).reshape(KW, n); i2 = u32(off_i2, n)
# check bucket ranges in buffer 1
def lt(a, b):
    for d in range(KW):
        if a[d] != b[d]: return a[d] < b[d]
    return False
bad = 0
for b in range(nb):
    lo, hi = bbase[b], bbase[b+1]
    for t in range(lo, hi):
        key = k1[:, t]
        if b > 0 and lt(key, split[:, b-1]): bad += 1
        if b < nb-1 and not lt(key, split[:, b]): bad += 1
print("bucket range violations", bad)
# indices are a permutation
print("i1 perm ok", np.array_equal(np.sort(i1 >> 2), np.arange(n)))
# leaf contents
allidx = []
for L in range(nl):
    bf, off, size, _ = desc[L]
    I = (i1 if bf == 1 else i2)[off:off+size]
    allidx.append(I >> 2)
allidx = np.concatenate(allidx)
print("leaf idx perm ok", np.array_equal(np.sort(allidx), np.arange(n)), len(allidx))
stat = u64(off_stat, maxl)[:nl]
print("status flags", np.bincount((stat >> np.uint64(62)).astype(int)), "last incl", int(stat[-1] & np.uint64((1<<62)-1)))
# which keys survive
xs, zs, ks, cs = [a[:int(cnt)] for a in (ox.cpu().numpy().view(np.uint64).T, oz.cpu().numpy().view(np.uint64).T, ok, oc)]
print("surviving coeffs", np.abs(oc[:int(cnt)].cpu().numpy())[:8])
