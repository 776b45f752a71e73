"""Top warp-stall SASS lines of an ncu report (diagnostic):
python scripts/ncu_top_sass.py report.ncu-rep [n] [kernel-section-index]

The source page lists one section per profiled launch ("Kernel Name" line,
then the header, then one row per SASS instruction)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
sec = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
for k, s in enumerate(starts):
    print(f"section {k}: {rows[s][1][:90]}")
s = starts[sec]
e = starts[sec + 1] if sec + 1 < len(starts) else len(rows)
h = rows[s + 1]
data = [r for r in rows[s + 2:e] if len(r) == len(h)]
ia, isrc = h.index("Address"), h.index("Source")
ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
num = lambda v: int(float(v or 0))
tot = sum(num(r[ss]) for r in data)
print("section", sec, "total stall samples", tot)
for i in sorted(range(len(data)), key=lambda i: -num(data[i][ss]))[:n]:
    r = data[i]
    print(f"== {r[ia][-5:]} {num(r[ss]) / tot:6.1%} exec {r[ie]:>8} {r[isrc][:70]}")
    for j in range(max(0, i - 2), i):
        print("        ", data[j][isrc][:80])
