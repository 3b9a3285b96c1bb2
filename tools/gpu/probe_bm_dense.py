"""K5 pipe choice on dense rows: 'direct' (INT/LOP3+POPC) vs 'tensor'
(tcgen05.mma.kind::i8) vs 'lists', uniform random strings (every qubit
uniform over I/X/Y/Z), M x M checks.  usage: python tools/gpu/probe_bm_dense.py [M]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))
import paper_2605_25974_b200 as pl  # noqa: E402
from paper_2605_25974_b200 import rng  # noqa: E402
from oracle import numpy_ref as R  # noqa: E402

dev = torch.device("cuda", 0)
M = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
for n in (500, 200, 100, 64):
    x, z, f, c = rng.random_columns(n, M, 11)
    S = pl.PauliSumSoA.from_columns(n, x, z, f, c, device=dev)
    res = {"n": n, "W": S.words, "M": M}
    outs = {}
    for meth in ("direct", "tensor", "lists"):
        try:
            out = pl.commutation_bitmatrix(S, method=meth)
            torch.cuda.synchronize()
            ms = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                pl.commutation_bitmatrix(S, method=meth, out=out)
                b.record()
                b.synchronize()
                ms.append(a.elapsed_time(b))
            outs[meth] = out
            t = min(ms)
            res[meth] = {"ms": round(t, 3), "checks_per_s": float(M) * M / (t / 1e3)}
        except Exception as e:  # noqa: BLE001
            res[meth] = {"error": str(e)[:120]}
    if "direct" in outs and "tensor" in outs:
        res["tensor_equals_direct"] = bool(torch.equal(outs["direct"], outs["tensor"]))
    if "tensor" in outs:
        rows = [0, 1, 127, 128, M // 2 + 5, M - 1]
        ok = True
        for r in rows:
            exp = R.pack_bitrows(R.bitmatrix(x, z, r, r + 1, 0, M))
            ok &= bool(np.array_equal(outs["tensor"][r:r + 1].cpu().numpy().view(np.uint32), exp))
        res["tensor_rows_vs_oracle"] = ok
    print(json.dumps(res), flush=True)
    del outs
    torch.cuda.empty_cache()
