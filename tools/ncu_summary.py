"""Summarise an ncu --set full capture (raw CSV page) into the metrics the
roofline in bench.py cites: per-launch DRAM bytes, duration, shared-memory
wavefronts / bank conflicts, issue utilisation.  Usage:
    python tools/ncu_summary.py gpurun_out/prof_raw.csv [kernel_label] [--traffic profiles/ncu_traffic.json]
"""
import csv
import json
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, units = rows[h], rows[h + 1]
    out = []
    for vals in rows[h + 2:]:
        if len(vals) != len(hdr):
            continue
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                j = hdr.index(k)
                try:
                    v = float(vals[j].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * SCALE.get(units[j], 1.0)
                d[k + ".unit"] = "s" if units[j] in ("ns", "us", "usecond", "ms", "msecond", "nsecond") else (
                    "B" if units[j].endswith("byte") else units[j])
        out.append(d)
    return out


def main():
    path = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
    res = load(path)
    for d in res:
        print(json.dumps(d, indent=1))
    if "--traffic" in sys.argv and label:
        tp = sys.argv[sys.argv.index("--traffic") + 1]
        try:
            t = json.load(open(tp))
        except FileNotFoundError:
            t = {}
        d = res[0]
        t[label] = {"dram_bytes_per_launch": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
                    "duration_s_under_ncu": d["gpu__time_duration.sum"],
                    "source": path.split("/")[-1], "kernel": d["kernel"]}
        json.dump(t, open(tp, "w"), indent=1)


if __name__ == "__main__":
    main()
