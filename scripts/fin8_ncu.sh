#!/bin/bash
# ncu launch list (time + DRAM bytes) of the final build's bench step.
OUT=gpurun_out/fin8; mkdir -p $OUT
EINET_LEAF_COND=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 260 -c 62 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --small-batch 0 > $OUT/launches.log 2>&1
echo "launches rc=$?" >> $OUT/status.txt
