#!/bin/bash
# C4 step time: session-start build (build_ab/lib_e11.so) vs the in-tree build.
set -u
OUT=gpurun_out/c4diag2; mkdir -p $OUT
run() { timeout 300 python bench.py --config C4 --batch $1 --chunk $1 --no-cpu-baseline --small-batch 0 --steps 20 > $OUT/c4.json 2>$OUT/err.txt
  python -c "
import json; d=json.load(open('$OUT/c4.json')); k=d['kernels']
print('$2', $1, round(d['ms_per_step']*1e3,1), {c: round(v['ms_per_step']*1e3,1) for c,v in k.items()})" >> $OUT/c4.txt; }
for r in 1 2; do for b in 1024 4096; do
  EINET_LIB_PATH=build_ab/lib_e11.so run $b e11
  run $b new
done; done
for r in 1 2; do
  EINET_LIB_PATH=build_ab/lib_e11.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > $OUT/c3.json 2>/dev/null
  python -c "import json; d=json.load(open('$OUT/c3.json')); print('c3 e11', round(d['ms_per_step']*1e3,1), [round(s['ms_per_step']*1e3,1) for s in d['secondary_batches']])" >> $OUT/c4.txt
  timeout 300 python bench.py --no-cpu-baseline --steps 50 > $OUT/c3.json 2>/dev/null
  python -c "import json; d=json.load(open('$OUT/c3.json')); print('c3 new', round(d['ms_per_step']*1e3,1), [round(s['ms_per_step']*1e3,1) for s in d['secondary_batches']])" >> $OUT/c4.txt
done
