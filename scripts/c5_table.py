"""Markdown table of a scripts/sweep_c5.py run (profiles/r02_c5_sweep.md):
python scripts/c5_table.py sweep.jsonl [single_term.jsonl]

The optional second file is a sweep run with EINET_CONTRACT_TERMS=1 (the
reduced-precision single-term forward); its forward time and algorithmic
tensor-core fraction are added as the last column."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1])]
one = {}
if len(sys.argv) > 2:
    for l in open(sys.argv[2]):
        d = json.loads(l)
        one[(d["k"], d["batch"])] = d
head = ("| K | B | bound | fwd us | fwd TF/s | fwd TC alg / issued | fwd HBM | W-stats us | "
        "W-stats TF/s (issued) | child-rho us | child-rho TF/s (issued) | prep us |")
sep = "|---" * 12 + "|"
if one:
    head += " fwd single-term us (TC alg) |"
    sep += "---|"
print(head)
print(sep)
for d in rows:
    line = (f"| {d['k']} | {d['batch']} | {d['bound']} | {d['fwd_us']:.1f} | {d['fwd_tflops']:.0f} | "
            f"{d['fwd_tc_frac']:.3f} / {d['fwd_tc_frac_issued'] or 0:.2f} | {d['fwd_hbm_frac']:.3f} | "
            f"{d['wstats_us']:.1f} | {d['wstats_tflops']:.0f} ({d['wstats_tc_frac_issued'] or 0:.2f}) | "
            f"{d['childrho_us']:.1f} | {d['childrho_tflops']:.0f} ({d['childrho_tc_frac_issued'] or 0:.2f}) | "
            f"{d['prep_us']:.1f} |")
    if one:
        o = one.get((d["k"], d["batch"]))
        line += f" {o['fwd_us']:.1f} ({o['fwd_tc_frac']:.3f}) |" if o else " |"
    print(line)
