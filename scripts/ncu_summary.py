"""Summarise ncu outputs into markdown for profiles/.

    python scripts/ncu_summary.py launches gpurun_out/TAG/launches.csv [steps]
    python scripts/ncu_summary.py full gpurun_out/TAG/full.ncu-rep
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path, steps=None):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        us = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
        n = d["Kernel Name"].split("(")[0]
        agg[n][0] += 1
        agg[n][1] += us
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total us | us/launch | share |", "|---|---|---|---|---|"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{n}` | {c} | {t:.1f} | {t / c:.1f} | {100 * t / tot:.1f}% |")
    out.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.1f} | | |")
    return "\n".join(out)


METRICS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "MB rd"),
    ("dram__bytes_write.sum", "MB wr"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", "hmma %"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ %"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units = r[0], r[1]
    idx = {n: i for i, n in enumerate(h)}
    out = ["| kernel | " + " | ".join(m[1] for m in METRICS) + " |",
           "|---|" + "---|" * len(METRICS)]
    for x in r[2:]:
        cells = []
        for m, _ in METRICS:
            i = idx.get(m)
            if i is None or x[i] == "":
                cells.append("-")
                continue
            v = float(x[i].replace(",", ""))
            u = units[i]
            if m.startswith("gpu__time"):
                v = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
            if m.startswith("dram__bytes"):
                v = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1) * v
            cells.append(f"{v:.1f}" if v < 1e4 else f"{v:.0f}")
        name = x[idx["Kernel Name"]].split("(")[0].replace("void ", "")
        out.append(f"| `{name}` | " + " | ".join(cells) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        print(full(sys.argv[2]))
