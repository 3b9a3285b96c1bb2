"""Aggregate ncu source-page samples (--print-source cuda,sass) by CUDA line.
usage: python tools/ncu_src_lines.py src.csv [function-substring] [topN]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
rows = list(csv.reader(open(path)))
fn = None
file = None
hdr = None
agg = defaultdict(lambda: [0, "", defaultdict(int)])
total = 0
for r in rows:
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
    if hdr is None or want not in (fn or ""):
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    s = int(r[4] or 0) if r[4].isdigit() else 0
    if s == 0:
        continue
    key = (file, line)
    agg[key][0] += s
    agg[key][1] = r[1].strip()[:90]
    for j, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                agg[key][2][h[6:]] += float(r[j] or 0)
            except ValueError:
                pass
    total += s
print("total samples", total)
for (f, l), (s, src, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    reasons = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    rs = " ".join(f"{k}={v / max(s, 1):.2f}" for k, v in reasons)
    print(f"{100 * s / total:5.1f}% {f}:{l:<5} {src:<70} {rs}")
