#!/usr/bin/env python
"""Benchmark: outer product + merge (pair-products/s) and commutation checks/s
at 500 qubits, on B200 (contract: see DESIGN.md "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline ``value``: BASELINE config 4 (two 10^4-term sums at n=500, weight 8
on qubits 0..47, seed 3 -> 10^8 pair products), multiply + merge through the
public API with device-resident inputs, whole-job pair-products/s over N GPUs
(strong scaling: the 10^8 products are split across ranks by B-term blocks,
key-range all-to-all over NCCL, local merge).  ``e2e`` is the same call with
host (pinned) input sums and the merged sum returned to host memory.
Secondary lines (N=1): config 2, config 1 batched multiply, config 5
bitmatrix / simplify / grouping.  The CPU baseline is the numpy restatement of
the reference (oracle/, "port") on a bounded sample, timed on this host.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "pair-products/s (outer product+merge) & commutation checks/s at 500 qubits"
UNIT = "pair-products/s"
WORKLOAD = ("C4: outer product + merge of two 10^4-term sums, n=500, weight 8 on qubits "
            "0..47, complex N(0,1) coefficients, seed 3 (10^8 pair products)")
L2_FLUSH_BYTES = 512 << 20


# kernels launched under one stage-timer entry of the native library
# (k_leaf_scan: the 3-kernel scan; k_regroup: prep, buckets, copy)
KERNELS_PER_STAGE = {"k_leaf_scan": 3, "k_regroup": 3}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def ncu_traffic(kernel: str):
    """Per-launch DRAM bytes of `kernel` from the committed ncu --set full summary."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        v = d.get(kernel)
        if isinstance(v, dict):
            return v.get("dram_bytes_per_launch")
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------- CPU side
CPU_SAMPLE_M = 3163          # 3163 x 3163 ~ 10^7 pair products per CPU step
C4_PRODUCTS = 10_000 * 10_000


def nlogn_scale(n_sample: int, n_full: int) -> float:
    """Time ratio T(n_full) / T(n_sample) for an n log n sort-and-merge
    (the CPU C4 baseline is timed at ~10^7 and extrapolated)."""
    import math

    return (n_full * math.log(n_full)) / (n_sample * math.log(n_sample))


def host_info() -> dict:
    info = {"cpu_count": os.cpu_count(), "affinity": None, "cpu_model": None, "ram_gb": None}
    try:
        info["affinity"] = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                info["ram_gb"] = round(int(line.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    return info


def cpu_outer_time(A, B, threads: int) -> float:
    """Seconds for the oracle restatement of sum_multiply (sums.py:293-305):
    multiply threaded over j-blocks (sums.py:158-173), combine single-threaded
    (sums.py:94-120), on the given prefix operands."""
    from oracle import numpy_ref as R

    t0 = time.perf_counter()
    R.outer_combine(*A, *B, threads=threads)
    return time.perf_counter() - t0


def cpu_sample_desc(m: int, threads: int) -> str:
    return (f"first {m} x {m} terms of the C4 inputs ({m * m} pair products) per step, time "
            f"extrapolated to the full 10^8 products as n log n (x{nlogn_scale(m * m, C4_PRODUCTS):.3f}, "
            f"BASELINE.md §3); multiply threaded over {threads} threads (sums.py:158-173), "
            f"combine single-threaded (sums.py:94-120); calibration: one full 10^8 run on this "
            f"pool's host took 85.8 s vs 80.9 s extrapolated (profiles/r2/cpu_c4_full.json)")


def run_reference(args, rank: int, world: int):
    """--impl reference: the reference's CPU algorithm (numpy port in oracle/;
    the reference is pure Python, nothing to compile) on this host's cores, on
    the C4 workload: each timed step is a ~10^7-product prefix sample whose
    time is extrapolated n log n to the 10^8-product step.  Warm-up steps use
    a 10^6-product prefix."""
    if rank != 0:
        return
    from paper_2605_25974_b200 import rng

    a, b = rng.config_columns(4)
    threads = os.cpu_count() or 1
    m = args.cpu_sample
    A = tuple(x[:m] for x in a)
    B = tuple(x[:m] for x in b)
    for _ in range(args.warmup):
        cpu_outer_time(tuple(x[:1000] for x in a), tuple(x[:1000] for x in b), threads)
    scale = nlogn_scale(m * m, C4_PRODUCTS)
    times = [cpu_outer_time(A, B, threads) * scale for _ in range(args.steps)]
    tot = sum(times)
    value = C4_PRODUCTS * len(times) / tot
    sample = cpu_sample_desc(m, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64+c128",
        "data": "synthetic (seeded SplitMix64 generator, DESIGN.md Inputs)",
        "config": {"workload": WORKLOAD, "pair_products_per_step": C4_PRODUCTS,
                   "sampled": sample, "extrapolated": "n log n from the timed sample",
                   "host": host_info()},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- launcher
def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-run this command as N ranks
    (one process per GPU) under torch.distributed.run on 127.0.0.1.  NCCL's
    INIT log goes to per-process files so rank 0 can report the communicator
    size NCCL itself saw."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", NCCL_LOG_PATTERN)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


NCCL_LOG_PATTERN = "/tmp/paulib_nccl.%h.%p.log"


def nccl_nranks() -> int | None:
    """nRanks of this process's NCCL communicator, from its INIT log (if any)."""
    import re
    import socket

    pat = os.environ.get("NCCL_DEBUG_FILE")
    if not pat:
        return None
    path = Path(pat.replace("%h", socket.gethostname()).replace("%p", str(os.getpid())))
    try:
        text = path.read_text(errors="replace")
    except OSError:
        return None
    found = re.findall(r"nRanks (\d+)", text) or re.findall(r"nranks (\d+)", text)
    return int(found[-1]) if found else None


# --------------------------------------------------------------- GPU side
def sum_bytes(s) -> int:
    m = len(s)
    return 2 * s.words * 8 * m + m + 16 * m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=CPU_SAMPLE_M)
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.launch_check:  # CPU test of the launcher: gloo rendezvous, no GPU work
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo")
        t = torch.tensor([rank + 1])
        dist.all_reduce(t)
        if rank == 0:
            print(json.dumps({"launch_check": True, "world": dist.get_world_size(),
                              "rank_sum": int(t.item())}), flush=True)
        dist.destroy_process_group()
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_25974_b200 as pl
    from paper_2605_25974_b200 import _native, rng

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    def barrier():
        if group is not None:
            dist.barrier(device_ids=[local])

    # ---- inputs (identical on every rank)
    a_cols, b_cols = rng.config_columns(4)
    A = pl.PauliSumSoA.from_columns(500, *a_cols, device=dev)
    B = pl.PauliSumSoA.from_columns(500, *b_cols, device=dev)
    n_items = len(A) * len(B)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    if world > 1:
        from paper_2605_25974_b200 import dist as pdist

        def step():
            return pdist.sharded_outer_multiply(A, B, group=group)
    else:
        def step():
            return pl.outer_multiply(A, B)

    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize()
    del out

    # ---- timed region: K steps, each bracketed by CUDA events on the stream
    stream = torch.cuda.current_stream(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    counts = []
    _native.stage_timing(True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)                    # evict L2 between steps
            evs[i][0].record(stream)
            out = step()
            evs[i][1].record(stream)
            counts.append(len(out))
            del out
        torch.cuda.synchronize()
    barrier()
    _native.stage_timing(False)
    stages = _native.stage_times()
    step_ms = [s.elapsed_time(e) for s, e in evs]
    tot_ms = sum(step_ms)
    if group is not None:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    value = n_items * args.steps / (tot_ms / 1e3)

    # roofline per pipeline kernel (algorithmic bytes per launch),
    # reported for the dominant one (largest share of the step)
    plan = pl.sums.LAST_PLAN or {}
    kw = plan.get("key_words", 2)
    hbm, peak_kind = measured_peaks()
    local_items = plan.get("n_items", n_items)
    local_out = counts[-1]
    item_b = 8 * kw + 4                       # packed key + ik
    ent_b = 8 * kw + 16                       # merged (key, sum) entry
    term_b = 16 * 8 + 1 + 16                  # SoA output term at W=8
    algo = {
        "k_count": (local_items * 2, "2 B bucket id written (items are generated, not read)"),
        "k_scatter": (local_items * (item_b + 2), f"2 B bucket id read + {item_b} B item written"),
        "k_split_count": (local_items * (8 * kw + 2),
                          f"{8 * kw} B item key read + 2 B sub-bucket id written"),
        "k_split_scatter": (local_items * (2 * item_b + 2),
                            f"{item_b} B item + 2 B sub-bucket id read, {item_b} B item written"),
        "k_leaf_sort": (local_items * item_b + local_out * ent_b,
                        f"{item_b} B item read + {ent_b} B (key, sum) per merged term written"),
        "k_emit": (local_out * (ent_b + term_b),
                   f"{ent_b} B (key, sum) read + {term_b} B SoA term written per merged term"),
    }
    per_kernel = {}
    for nm, (bts, desc) in algo.items():
        ms = [m for k2, m in stages if k2 == nm]
        if not ms:
            continue
        avg = statistics.mean(ms) / 1e3
        ach = bts / avg / 1e9
        per_kernel[nm] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                          "frac": ach / hbm, "avg_launch_ms": avg * 1e3,
                          "algorithmic_bytes_per_launch": bts, "bytes_per_unit": desc,
                          "traffic": ncu_traffic(nm)}
    roofline = None
    if per_kernel:
        dom = max(per_kernel, key=lambda k2: per_kernel[k2]["avg_launch_ms"])
        roofline = dict(per_kernel[dom], kernel=dom, peak_source=peak_kind)
        step_bytes = local_out * term_b + sum_bytes(A) + sum_bytes(B)
        step_s = (tot_ms / args.steps) / 1e3
        roofline["step"] = {"algorithmic_bytes": step_bytes,
                            "bytes_per_unit": f"{term_b} B output term + operands read",
                            "achieved": step_bytes / step_s / 1e9,
                            "frac": step_bytes / step_s / 1e9 / hbm}
        roofline["kernels"] = per_kernel
    stage_share = {}
    for nm, ms in stages:
        stage_share[nm] = stage_share.get(nm, 0.0) + ms
    stage_share = {k: round(v / max(tot_ms, 1e-9), 4) for k, v in stage_share.items()}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        Ah = A.cpu()
        Bh = B.cpu()
        Ah = pl.PauliSumSoA(500, Ah.x.pin_memory(), Ah.z.pin_memory(), Ah.flags.pin_memory(),
                            Ah.coeffs.pin_memory(), validate=False)
        Bh = pl.PauliSumSoA(500, Bh.x.pin_memory(), Bh.z.pin_memory(), Bh.flags.pin_memory(),
                            Bh.coeffs.pin_memory(), validate=False)

        def e2e_step():
            if world > 1:
                return pdist.sharded_outer_multiply(Ah, Bh, group=group, device=dev)
            return pl.sum_multiply(Ah, Bh)

        r = e2e_step()                                   # warm-up (pinned pools)
        # bytes actually copied: planes that are zero in every operand are
        # cleared on the host instead of crossing PCIe (sums._download)
        d2h = int(pl.sums.LAST_D2H_BYTES)
        result_bytes = sum_bytes(r)
        del r
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ne = max(1, min(args.steps, 3))
        for _ in range(ne):
            r = e2e_step()
            del r
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if group is not None:
            t = torch.tensor([el], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": n_items * ne / el, "unit": UNIT,
               "h2d_bytes_per_step": sum_bytes(A) + sum_bytes(B), "d2h_bytes_per_step": d2h,
               "host_result_bytes_per_step": result_bytes,
               "ms_per_step": 1e3 * el / ne}

    # ---- CPU baseline and secondary workloads (rank 0 at N=1 only)
    cpu = None
    secondary = {}
    if world == 1 and rank == 0:
        if not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            m = args.cpu_sample
            sec = cpu_outer_time(tuple(x[:m] for x in a_cols), tuple(x[:m] for x in b_cols),
                                 threads)
            t_full = sec * nlogn_scale(m * m, C4_PRODUCTS)
            cpu = {"value": C4_PRODUCTS / t_full, "unit": UNIT, "cores": threads, "kind": "port",
                   "sample": cpu_sample_desc(m, threads) + f"; one run, {sec:.2f} s",
                   "host": host_info()}
        if not args.no_secondary:
            from bench_secondary import run_secondary

            secondary = run_secondary(dev, flush)
    elif world > 1 and not args.no_secondary:
        from bench_secondary import c5_bitmatrix_sharded

        secondary = c5_bitmatrix_sharded(dev, flush, group)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u64+c128", "data": "synthetic (seeded SplitMix64 generator, DESIGN.md Inputs)",
            "config": {"workload": WORKLOAD, "pair_products_per_step": n_items,
                       "merged_terms": counts[-1] if counts else None,
                       "l2": "512 MiB buffer written between timed steps; working set >> L2",
                       "key_words": kw, "buckets": plan.get("n_buckets")},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": sum(KERNELS_PER_STAGE.get(nm, 1) for nm, _ in stages),
            "clocks": clk.summary(), "stage_share": stage_share,
            "nccl_nranks": nccl_nranks() if world > 1 else None,
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
