"""Top warp-stall SASS lines of an ncu report (diagnostic): python
scripts/ncu_top_sass.py report.ncu-rep [n]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = rows[2:]
ia, isrc = h.index("Address"), h.index("Source")
ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ss] or 0) for r in data)
print("total stall samples", tot)
for i in sorted(range(len(data)), key=lambda i: -int(data[i][ss] or 0))[:n]:
    r = data[i]
    print(f"== {r[ia][-5:]} {int(r[ss] or 0) / tot:6.1%} exec {r[ie]:>8} {r[isrc][:70]}")
    for j in range(max(0, i - 2), i):
        print("        ", data[j][isrc][:80])
