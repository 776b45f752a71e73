#!/bin/bash
OUT=gpurun_out/e2erep; mkdir -p $OUT
for r in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline --small-batch 0 --steps 100 > $OUT/b$r.json 2>/dev/null
  python -c "
import json; d=json.load(open('$OUT/b$r.json')); e=d['e2e']
print(round(d['ms_per_step']*1e3,1), round(e['value']/1e6,2), round(e['h2d_gbs'],1), round(e['h2d_link_gbs'],1), round(e['fp32_host_input']['value']/1e6,2), round(e['f64_numpy_input']['value']/1e6,2))" >> $OUT/e2e.txt
done
