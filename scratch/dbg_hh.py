import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
from conftest import golden
import paper_2605_25974_b200 as pl
from oracle import numpy_ref as R
dev = torch.device('cuda')
g = golden("outer_hh")
h = pl.PauliSumSoA.from_columns(64, g["hx"], g["hz"], g["hf"], g["hc"], device=dev)
out = h * h
x, z, k, c = out.columns()
print("got", len(out), "exp", len(g["ox"]))
# uniqueness / sortedness
keys = np.stack([z[:, 0], x[:, 0]], 1)
ek = np.stack([g["oz"][:, 0], g["ox"][:, 0]], 1)
print("unique got", len(np.unique(keys, axis=0)), "sorted:", all(tuple(keys[i]) < tuple(keys[i+1]) for i in range(len(keys)-1)))
s_got = set(map(tuple, keys.tolist())); s_exp = set(map(tuple, ek.tolist()))
print("missing", len(s_exp - s_got), "extra", len(s_got - s_exp))
raw = pl.sum_multiply(h, h, combine=False)
rx, rz, rk, rc = raw.columns()
ex = R.combine(rx, rz, rk, rc)
print("oracle on gpu-raw", len(ex[0]))
print(list(s_exp - s_got)[:5])
# plan info
import ctypes as C
from paper_2605_25974_b200 import _native
from paper_2605_25974_b200._device import ptr, stream_ptr
A = h.planes()
plan = _native.MergePlan()
_native.call("pl_outer_plan", 1, 60, 60, ptr(A.x), ptr(A.z), A.ld, ptr(A.x), ptr(A.z), A.ld, C.byref(plan), stream_ptr(dev))
print("KW", plan.key_words, "bits", plan.key_bits, "nb", plan.n_buckets, "cap", plan.leaf_cap, list(plan.seg_lo)[:2], list(plan.seg_len)[:2], list(plan.seg_pos)[:2], plan.reserved[0])
