"""Exactness of K6 on a long prefix of config 5 against the C oracle
(first-fit is prefix-closed).  usage: python tools/gpu/check_c5_group_prefix.py [terms]"""
import sys, time
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[2]))
import numpy as np, torch
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng
from oracle import cgreedy
m = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
x, z, f, c = rng.c5_columns(1_000_000)
x, z, f, c = x[:m], z[:m], f[:m], c[:m]
t0 = time.time(); gof, ng, pc = cgreedy.greedy(x, z); t1 = time.time()
S = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=torch.device('cuda', 0))
g, n, p = pl.group_assignment(S)
g = g.cpu().numpy()
print('oracle %.1f s groups %d checks %d | gpu groups %d checks %d | equal assignment %s equal checks %s'
      % (t1 - t0, ng, pc, int(n.item()), int(p.item()), bool(np.array_equal(g, np.asarray(gof))), int(p.item()) == pc))
