"""Print the headline numbers and per-kernel-class split of a bench.py JSON line."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"value {d['value']:.4g} {d['unit']}  ms/step {d['ms_per_step']:.4f}  e2e {d['e2e']['value']:.4g}"
      f"  launches {d.get('gpu_launches')}  clocks {d.get('clocks')}")
print("roofline", d.get("roofline"))
print("cpu", d.get("cpu_baseline"))
tot = 0
for k, v in d.get("kernels", {}).items():
    tot += v["ms_per_step"]
    print(f"  {k:18s} {1e3 * v['ms_per_step']:8.1f} us  share {v['share']:.3f}  tflops {v['tflops']}")
print(f"  sum {1e3 * tot:.1f} us")
