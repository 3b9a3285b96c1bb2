"""One full-size CPU run of the C4 workload (10^8 pair products) with the
oracle port of sum_multiply (multiply threaded over all cores, combine
single-threaded, as the reference), next to the 10^7-product sample the bench
extrapolates from -- calibrates bench.py's n log n extrapolation.  Needs ~60 GB
of host RAM.  usage: python tools/cpu_c4_full.py > profiles/r2/cpu_c4_full.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from bench import C4_PRODUCTS, CPU_SAMPLE_M, host_info, nlogn_scale  # noqa: E402
from oracle import numpy_ref as R  # noqa: E402
from paper_2605_25974_b200 import rng  # noqa: E402

a, b = rng.config_columns(4)
threads = os.cpu_count() or 1
m = CPU_SAMPLE_M
t0 = time.perf_counter()
R.outer_combine(*(v[:m] for v in a), *(v[:m] for v in b), threads=threads)
t_sample = time.perf_counter() - t0
t0 = time.perf_counter()
out = R.outer_combine(*a, *b, threads=threads)
t_full = time.perf_counter() - t0
print(json.dumps({
    "what": "C4 on the CPU (oracle port of sum_multiply: multiply threaded, combine single-threaded)",
    "threads": threads, "host": host_info(),
    "sample_products": m * m, "sample_s": t_sample,
    "extrapolated_full_s": t_sample * nlogn_scale(m * m, C4_PRODUCTS),
    "full_products": C4_PRODUCTS, "full_s": t_full, "merged_terms": int(out[0].shape[0]),
    "full_pair_products_per_s": C4_PRODUCTS / t_full}))
