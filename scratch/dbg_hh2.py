import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
from conftest import golden
import paper_2605_25974_b200 as pl
from oracle import numpy_ref as R
dev = torch.device('cuda')
g = golden("outer_hh")
h = (g["hx"], g["hz"], g["hf"], g["hc"])
print([a.dtype for a in h], [a.shape for a in h], h[0][:3].ravel(), h[1][:3].ravel())
A = pl.PauliSumSoA.from_columns(64, *h, device=dev)
print(A.x[:, :3], A.z[:, :3])
raw = pl.sum_multiply(A, A, combine=False)
rx, rz, rk, rc = raw.columns()
ex, ez, ek, ec = R.outer_raw(*h, *h)
bad = np.flatnonzero((rx[:, 0] != ex[:, 0]) | (rz[:, 0] != ez[:, 0]) | (rk != ek))
print("bad rows", len(bad), bad[:10])
for r in bad[:3]:
    print(r, rx[r], ex[r], rz[r], ez[r], rk[r], ek[r])
print("coef maxdiff", np.abs(rc - ec).max())
