#!/bin/bash
# W statistics per cluster size (EINET_WS_NCL cap): C3 per-class times at three batches
OUT=gpurun_out/${1:-wsncl}; mkdir -p $OUT
for ncl in 1 2 4; do
  for b in 16384 4096 500; do
    r=$(EINET_WS_NCL=$ncl timeout 120 python scripts/class_times.py C3 $b 2>&1 | tail -1)
    echo "ncl=$ncl B=$b $r" >> $OUT/ncl.txt
  done
done
