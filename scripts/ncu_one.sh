#!/bin/bash
# ncu --set full of one kernel (regex $2) in the C3 bench step, into gpurun_out/$1
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
EINET_LEAF_COND=0 timeout 900 ncu --set full --clock-control none --import-source on -s ${SKIP:-40} -c ${COUNT:-1} \
  -k "regex:$2" -o $OUT/full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --small-batch 0 > $OUT/full.log 2>&1
echo "ncu rc=$?" >> $OUT/status.txt
