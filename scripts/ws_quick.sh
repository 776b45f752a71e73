#!/bin/bash
# W statistics class times on C3 (three batches), optional env in $WSENV
OUT=gpurun_out/${1:-wsq}; mkdir -p $OUT
for b in 16384 4096 500; do
  r=$(env $WSENV timeout 120 python scripts/class_times.py C3 $b 2>/dev/null | tail -1)
  echo "$WSENV B=$b $r" >> $OUT/q.txt
done
