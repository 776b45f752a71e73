#!/bin/bash
# C4 step time: build_ab/lib_b49.so (before the leaf-statistics changes) vs the in-tree build.
set -u
OUT=gpurun_out/c4diag3; mkdir -p $OUT
run() { timeout 300 python bench.py --config C4 --batch $1 --chunk $1 --no-cpu-baseline --small-batch 0 --steps 20 > $OUT/c4_$2_$1.json 2>$OUT/err_$2_$1.txt
  python -c "
import json; d=json.load(open('$OUT/c4_$2_$1.json')); k=d['kernels']
print('$2', $1, round(d['ms_per_step']*1e3,1), {c: round(v['ms_per_step']*1e3,1) for c,v in k.items()})" >> $OUT/c4.txt; }
for r in 1 2; do for b in 1024 4096; do
  EINET_LIB_PATH=build_ab/lib_b49.so run $b b49
  run $b new
done; done
