"""profiles/kernel_traffic.json from an ncu launch list with DRAM metrics
(`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`):
per kernel, the DRAM read + write bytes of every launch (the bench line's
`roofline.traffic`).

    python scripts/kernel_traffic.py gpurun_out/TAG/launches.csv SOURCE-NOTE
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    path, note = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("einet::", "")
        per[(name, d["ID"])][d["Metric Name"]] += (float(d["Metric Value"].replace(",", ""))
                                                   * UNIT.get(d["Metric Unit"], 1))
    out = collections.defaultdict(list)
    for (name, _), m in per.items():
        out[name].append(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
    doc = {n: {"dram_bytes_per_launch": v, "source": note} for n, v in sorted(out.items())}
    with open(os.path.join(ROOT, "profiles", "kernel_traffic.json"), "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps({n: max(v["dram_bytes_per_launch"]) for n, v in doc.items()}, indent=1))


if __name__ == "__main__":
    main()
