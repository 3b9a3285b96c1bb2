import sys; sys.path.insert(0, ".")
import torch, numpy as np
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng
from oracle import numpy_ref as R
dev = torch.device("cuda", 0)
for m in (1, 10, 1000, 5000):
    x, z, f, c = rng.random_columns(20, m, 3)
    s = pl.PauliSumSoA.from_columns(20, x, z, f, c, device=dev)
    out = pl.sort_combine(s)
    ex = R.combine(x, z, f, c)
    ox = out.columns()[0]
    print(m, len(out), len(ex[0]), ox.shape == ex[0].shape and np.array_equal(ox, ex[0]), flush=True)
