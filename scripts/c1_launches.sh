#!/bin/bash
OUT=gpurun_out/c1l; mkdir -p $OUT
EINET_LEAF_COND=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 50 --csv \
  --log-file $OUT/c1.csv python bench.py --config C1 --batch 100 --chunk 100 --no-cpu-baseline --small-batch 0 --steps 2 --warmup 3 > $OUT/c1.log 2>&1
EINET_LEAF_COND=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 50 --csv \
  --log-file $OUT/c2.csv python bench.py --config C2 --batch 100 --chunk 100 --no-cpu-baseline --small-batch 0 --steps 2 --warmup 3 > $OUT/c2.log 2>&1
