"""C5 greedy grouping (10^6 terms, n=500) on growing prefixes: time, groups,
reference pair_checks.  usage: python tools/gpu/probe_c5_group.py [max_terms]"""
import sys
import time

import torch

sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))
import paper_2605_25974_b200 as pl  # noqa: E402
from paper_2605_25974_b200 import rng  # noqa: E402

dev = torch.device("cuda", 0)
top = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
x, z, f, c = rng.c5_columns(1_000_000)
for m in (20_000, 100_000, 300_000, 1_000_000):
    if m > top:
        break
    S = pl.PauliSumSoA.from_columns(500, x[:m], z[:m], f[:m], c[:m], device=dev)
    for it in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gof, ng, pc = pl.group_assignment(S)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"m={m} it={it} {dt * 1e3:.1f} ms groups={int(ng.item())} pair_checks={int(pc.item())} "
              f"checks/s={int(pc.item()) / dt:.3e}", flush=True)
