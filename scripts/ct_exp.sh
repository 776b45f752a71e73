#!/bin/bash
# contraction experiments: class times under EINET_CT_DEBUG / EINET_CT_G variants
OUT=gpurun_out/${1:-ctexp}; mkdir -p $OUT
for g in ${GS:-1 2}; do for d in ${DS:-0 1 2 4 5}; do
  echo "G=$g debug=$d $(EINET_CT_G=$g EINET_CT_DEBUG=$d python scripts/class_times.py 2>&1 | tail -1)" >> $OUT/exp.txt
done; done
