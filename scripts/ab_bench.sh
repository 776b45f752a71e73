#!/bin/bash
# A/B bench step times (graph replay, no CPU legs) of two builds on one box:
#   scripts/ab_bench.sh TAG other.so
OUT=gpurun_out/$1; mkdir -p $OUT
for r in 1 2; do for lib in "" "$2"; do
  EINET_LIB_PATH=${lib:-paper_2004_06231_b200/libeinet_b200.so} timeout 300 python bench.py --no-cpu-baseline --steps 50 > $OUT/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('$OUT/b.json'))
print('${lib:-new}'[-20:], round(d['ms_per_step']*1e3,1), [round(s['ms_per_step']*1e3,1) for s in d['secondary_batches']])" >> $OUT/ab.txt
done; done
