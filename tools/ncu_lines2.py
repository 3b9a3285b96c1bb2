"""Per-CUDA-line warp instructions and stall samples of one kernel from an
ncu source page exported with --print-source cuda,sass.
usage: python tools/ncu_lines2.py src.csv kernel-substring [topN]"""
import csv
import sys
from collections import defaultdict

path, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fn = file = hdr = None
agg = defaultdict(lambda: [0.0, 0.0, ""])
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or want not in (fn or "") or not r[0].isdigit():
        continue
    try:
        samp, inst = float(r[4]), float(r[7])
    except (ValueError, IndexError):
        continue
    a = agg[(file, int(r[0]))]
    a[0] += inst
    a[1] += samp
    a[2] = r[1][:100]
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"{want}: {ti / 1e6:.0f}M warp instructions, {ts:.0f} stall samples")
for k, v in sorted(agg.items(), key=lambda kv: -(kv[1][0] / ti + kv[1][1] / ts))[:top]:
    print(f"{100 * v[0] / ti:5.1f}% inst {100 * v[1] / ts:5.1f}% samp  {k[0]}:{k[1]}  {v[2]}")
