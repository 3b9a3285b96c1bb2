"""Secondary bench lines (N=1): the other BASELINE configs on the same B200.

Each entry: {"value", "unit", "ms_per_step", ...} timed with CUDA events on the
launching stream after warm-up, L2 flushed between timed repetitions.
"""

from __future__ import annotations

import json
import statistics
from pathlib import Path

import numpy as np
import torch

import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import _native, rng

ROOT = Path(__file__).resolve().parent


def _hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text()).get("hbm_gbs", 6650.0)) if p.exists() else 6650.0


def _timed(fn, dev, flush, reps: int, warm: int = 2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream(dev)
    ms = []
    for i in range(reps):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return ms


def c2(dev, flush):
    a, b = rng.config_columns(2)
    A = pl.PauliSumSoA.from_columns(500, *a, device=dev)
    B = pl.PauliSumSoA.from_columns(500, *b, device=dev)
    ms = _timed(lambda: pl.outer_multiply(A, B), dev, flush, 10)
    t = statistics.mean(ms)
    return {"workload": "C2: 1000 x 1000 outer product + merge, 4-local on qubits 0..23, seed 1",
            "value": 1e6 / (t / 1e3), "unit": "pair-products/s", "ms_per_step": t}


def c1(dev, flush):
    out = {}
    for P, label in ((65536, "C1: 65,536 pairs, n=500, seed 0/1"),
                     (1 << 24, "C1 shape at P=2^24 (HBM roofline check)")):
        a = rng.random_columns(500, min(P, 65536), 0)
        b = rng.random_columns(500, min(P, 65536), 1)
        reps_p = P // min(P, 65536)
        ax = torch.from_numpy(np.ascontiguousarray(np.tile(a[0].T, (1, reps_p))).view(np.int64)).to(dev)
        az = torch.from_numpy(np.ascontiguousarray(np.tile(a[1].T, (1, reps_p))).view(np.int64)).to(dev)
        bx = torch.from_numpy(np.ascontiguousarray(np.tile(b[0].T, (1, reps_p))).view(np.int64)).to(dev)
        bz = torch.from_numpy(np.ascontiguousarray(np.tile(b[1].T, (1, reps_p))).view(np.int64)).to(dev)
        ak = torch.zeros(P, dtype=torch.uint8, device=dev)
        bk = torch.zeros(P, dtype=torch.uint8, device=dev)
        inner = 200 if P <= 65536 else 5

        def run():
            for _ in range(inner):
                pl.batch_multiply(ax, az, ak, bx, bz, bk)

        # the launches are captured once in a CUDA graph and replayed
        # (SURVEY hard part 6: no Python/ctypes dispatch in the timed loop)
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            run()
        torch.cuda.current_stream(dev).wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            run()
        ms = _timed(graph.replay, dev, flush, 5)
        t = statistics.mean(ms) / inner
        pairs = P / (t / 1e3)
        gbs = 387 * P / (t / 1e3) / 1e9
        out["c1" if P == 65536 else "c1_2e24"] = {
            "workload": label, "value": pairs, "unit": "pairs/s", "ms_per_launch": t,
            "timing": f"CUDA graph of {inner} launches, replayed",
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": _hbm(), "unit": "GB/s",
                         "frac": gbs / _hbm(), "bytes_per_unit": "387 B/pair (W=8)"}}
    return out


def c5(dev, flush):
    x, z, f, c = rng.c5_columns(1_000_000, seed=4)
    S = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=dev)
    M = len(S)
    res = {}
    # simplify
    ms = _timed(lambda: pl.sort_combine(S), dev, flush, 5)
    t = statistics.mean(ms)
    res["c5_simplify"] = {"workload": "C5 sort_and_combine, 10^6 terms, seed 4",
                          "value": M / (t / 1e3), "unit": "terms/s", "ms_per_step": t,
                          "merged_terms": len(pl.sort_combine(S))}
    # full commutation bitmatrix, row chunks into one reused output buffer
    rows = 65536
    nw = (M + 31) // 32
    buf = torch.empty((rows, nw), dtype=torch.int32, device=dev)

    def bitmatrix():
        for r0 in range(0, M, rows):
            r = min(rows, M - r0)
            pl.commutation_bitmatrix(S, row0=r0, rows=r, out=buf[:r])

    _native.stage_timing(True)
    ms = _timed(bitmatrix, dev, flush, 2, warm=1)
    _native.stage_timing(False)
    st = _native.stage_times()
    kms = [m for n, m in st if n.startswith("k_bitmatrix")]
    t = statistics.mean(ms)
    checks = float(M) * M
    out_bytes = M * nw * 4
    # dominant kernel: bytes = 1 bit per check written (+ its row lists), vs HBM peak
    kt = sum(kms) / max(len(ms) + 1, 1) if kms else None
    res["c5_bitmatrix"] = {
        "workload": "C5 full commutation bitmatrix 10^6 x 10^6 (row chunks of 65536)",
        "value": checks / (t / 1e3), "unit": "checks/s", "ms_per_step": t,
        "output_bytes": out_bytes,
        "roofline": {"bound": "hbm", "achieved": out_bytes / (t / 1e3) / 1e9, "peak": _hbm(),
                     "unit": "GB/s", "frac": out_bytes / (t / 1e3) / 1e9 / _hbm(),
                     "bytes_per_unit": "1 bit written per check"},
    }
    return res


def c3(dev, flush):
    x, z, f, c = rng.config_columns(3)
    S = pl.PauliSumSoA.from_columns(100, x, z, f, c, device=dev)
    try:
        gof, ng, pc = pl.group_assignment(S)
    except _native.NativeLibraryError as e:
        return {"c3_grouping": {"skipped": str(e)[:120]}}
    ms = _timed(lambda: pl.group_assignment(S), dev, flush, 2, warm=1)
    t = statistics.mean(ms)
    checks = int(pc.item())
    return {"c3_grouping": {"workload": "C3 greedy grouping, JW-style n=100, 10^5 terms, seed 2",
                            "value": checks / (t / 1e3), "unit": "reference pair_checks/s",
                            "ms_per_step": t, "groups": int(ng.item()), "pair_checks": checks}}


def c5_grouping(dev, flush):
    """Config 5 greedy grouping at its full size (10^6 terms, n=500, W=8)."""
    x, z, f, c = rng.c5_columns(1_000_000, seed=4)
    S = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=dev)
    gof, ng, pc = pl.group_assignment(S)
    ms = _timed(lambda: pl.group_assignment(S), dev, flush, 2, warm=1)
    t = statistics.mean(ms)
    checks = int(pc.item())
    return {"c5_grouping": {"workload": "C5 greedy grouping, 10^6 terms n=500, seed 4",
                            "value": checks / (t / 1e3), "unit": "reference pair_checks/s",
                            "ms_per_step": t, "groups": int(ng.item()), "pair_checks": checks}}


TC_I8_PEAK = 4.5345e15  # tools/microbench/tc_i8.cu on this pool's B200 (profiles/r2/bitmatrix_pipes.json)


def dense_bitmatrix(dev, flush):
    """K5 on dense rows (uniform random strings, n=500, 65,536 x 65,536 checks):
    'auto' takes the tcgen05 int8 path; the INT 'direct' path beside it."""
    M = 65536
    x, z, f, c = rng.random_columns(500, M, 11)
    S = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=dev)
    out = torch.empty((M, M // 32), dtype=torch.int32, device=dev)
    res = {}
    for meth in ("auto", "direct"):
        ms = _timed(lambda: pl.commutation_bitmatrix(S, method=meth, out=out), dev, flush, 3)
        t = statistics.mean(ms)
        checks = float(M) * M
        line = {"workload": f"K5 dense bitmatrix, uniform random n=500, {M} x {M}, method {meth}",
                "value": checks / (t / 1e3), "unit": "checks/s", "ms_per_step": t}
        if meth == "auto":
            ops = checks * 2 * 128 * 8 / (t / 1e3)
            line["roofline"] = {"bound": "tensor", "achieved": ops / 1e12, "peak": TC_I8_PEAK / 1e12,
                                "unit": "TOP/s (int8)", "frac": ops / TC_I8_PEAK,
                                "bytes_per_unit": "2K = 2048 int8 ops per check (K = 128 W)"}
        else:
            lop = checks * 34 / (t / 1e3)
            line["roofline"] = {"bound": "int", "achieved": lop / 1e12, "peak": 18.375,
                                "unit": "T LOP3/s", "frac": lop / 18.375e12,
                                "bytes_per_unit": "~34 LOP3 + 1 POPC per check (W=8)"}
        res["k5_dense_" + meth] = line
    return res


def f3(dev, flush):
    """§8(f) row f3: two-phase parallel grouping of config 3 (8 chunks); the
    partition differs from the sequential greedy one by design, so the group
    count divergence is reported (bench.py:255-262 of the reference)."""
    x, z, f, c = rng.config_columns(3)
    S = pl.PauliSumSoA.from_columns(100, x, z, f, c, device=dev)
    st = pl.GroupingStats()
    part = pl.group_greedy_parallel(S, 8, stats=st)
    ms = _timed(lambda: pl.group_greedy_parallel(S, 8), dev, flush, 2, warm=1)
    t = statistics.mean(ms)
    _, ng, _ = pl.group_assignment(S)
    return {"f3_grouping_parallel": {
        "workload": "f3 group_greedy_parallel, C3 (JW n=100, 10^5 terms), 8 chunks",
        "value": st.pair_checks / (t / 1e3), "unit": "reference pair_checks/s", "ms_per_step": t,
        "groups": part.group_count(), "groups_sequential_greedy": int(ng.item()),
        "pair_checks": st.pair_checks}}


def f12(dev, flush):
    """§8(f) rows: Clifford gates (f2) and the rotation split + merge (f1) on
    C5-style sums (n=500, W=8), 2^24 terms for the gates (HBM roofline), 2^21
    for the rotation."""
    out = {}
    M = 1 << 24
    x, z, f, c = rng.random_columns(500, 1 << 16, 41)
    S = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=dev)
    # tile the 2^16 drawn terms to 2^24 on the device (content is irrelevant to timing)
    S.x = S.x.repeat(1, M >> 16).contiguous()
    S.z = S.z.repeat(1, M >> 16).contiguous()
    S.flags = S.flags.repeat(M >> 16).contiguous()
    S.coeffs = S.coeffs.repeat(M >> 16).contiguous()
    # algorithmic bytes per term: H reads x, z, phase of one word (17 B) and
    # writes x, z (16 B) + the phase of Y terms (1/4); CNOT across two words
    # reads 4 words + phase (33 B), writes x_t, z_c (16 B) + flipped phases (1/8)
    for gate, q, bpt in (("H", 77, 33.25), ("CNOT", (3, 300), 49.125)):
        ms = _timed(lambda: S.apply_clifford(gate, q), dev, flush, 10)
        t = statistics.mean(ms)
        byts = M * bpt
        out[f"f2_clifford_{gate}"] = {
            "workload": f"f2 apply_clifford {gate} on 2^24 terms, n=500",
            "value": M / (t / 1e3), "unit": "terms/s", "ms_per_step": t,
            "roofline": {"bound": "hbm", "achieved": byts / (t / 1e3) / 1e9, "peak": _hbm(),
                         "unit": "GB/s", "frac": byts / (t / 1e3) / 1e9 / _hbm(),
                         "bytes_per_unit": f"{bpt} B (touched words + phase, read + written)"}}
    del S
    torch.cuda.empty_cache()
    # Pauli-propagation-like inputs: config-5 style terms (weight 2-12 over
    # 500 qubits) and a sparse generator
    m = 1 << 21
    x, z, f, c = rng.c5_columns(m, seed=42)
    S = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=dev)
    gx, gz, _, _ = rng.c5_columns(1, seed=43)
    rot = pl.RotationSpec(pl.PauliString(500, gx[0], gz[0], 0), 0.37)
    raw = S.apply_rotation(rot, combine=False)
    mo = len(raw)
    del raw
    ms = _timed(lambda: S.apply_rotation(rot, combine=False), dev, flush, 10)
    t = statistics.mean(ms)
    byts = m * (145 + 8) + mo * 145  # read terms + anti/scan words, write split terms
    out["f1_rotation_split"] = {
        "workload": "f1 rotation split (un-combined), 2^21 C5-style terms n=500, sparse generator",
        "value": m / (t / 1e3), "unit": "input terms/s", "ms_per_step": t, "output_terms": mo,
        "roofline": {"bound": "hbm", "achieved": byts / (t / 1e3) / 1e9, "peak": _hbm(),
                     "unit": "GB/s", "frac": byts / (t / 1e3) / 1e9 / _hbm(),
                     "bytes_per_unit": "145 B term read + 8 B flags/scan + 145 B per output term"}}
    ms = _timed(lambda: S.apply_rotation(rot), dev, flush, 5)
    t = statistics.mean(ms)
    out["f1_apply_rotation"] = {
        "workload": "f1 apply_rotation (split + sort_and_combine), 2^21 C5-style terms n=500",
        "value": m / (t / 1e3), "unit": "input terms/s", "ms_per_step": t}
    return out


def c5_bitmatrix_sharded(dev, flush, group) -> dict:
    """N>1: the C5 commutation bitmatrix row-sharded over the ranks (north
    star: row blocks, inputs replicated, no collective).  Each rank computes
    rows [r*M/G, (r+1)*M/G) in 65,536-row chunks; whole-job checks/s = M^2 /
    the slowest rank's time."""
    import torch.distributed as dist

    from paper_2605_25974_b200 import dist as pdist

    x, z, f, c = rng.c5_columns(1_000_000, seed=4)
    S = pl.PauliSumSoA.from_columns(500, x, z, f, c, device=dev)
    M = len(S)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    r0, r1 = pdist.block_range(M, world, rank)
    rows = 65536
    nw = (M + 31) // 32
    buf = torch.empty((rows, nw), dtype=torch.int32, device=dev)

    def shard():
        for q0 in range(r0, r1, rows):
            r = min(rows, r1 - q0)
            pl.commutation_bitmatrix(S, row0=q0, rows=r, out=buf[:r])

    dist.barrier(group, device_ids=[dev.index])
    ms = _timed(shard, dev, flush, 2, warm=1)
    t = torch.tensor([statistics.mean(ms)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    t = float(t.item())
    out_bytes = M * nw * 4
    return {"c5_bitmatrix_sharded": {
        "workload": f"C5 full commutation bitmatrix 10^6 x 10^6, row blocks over {world} GPUs",
        "value": float(M) * M / (t / 1e3), "unit": "checks/s", "ms_per_step": t,
        "scaling": "strong", "n_gpus": world, "output_bytes": out_bytes,
        "timing": "CUDA events per rank, max over ranks"}}


def run_secondary(dev, flush) -> dict:
    out = {}
    for fn in (c2, c1, c5, c3, c5_grouping, dense_bitmatrix, f12, f3):
        try:
            r = fn(dev, flush)
        except Exception as e:  # keep the headline line even if a side metric fails
            r = {fn.__name__: {"error": f"{type(e).__name__}: {e}"[:200]}}
        if "workload" in r:
            out[fn.__name__] = r
        else:
            out.update(r)
        torch.cuda.empty_cache()
    return out
