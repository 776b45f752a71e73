#!/bin/bash
# A/B per-class times of two library builds on the same box (diagnostics):
#   scripts/ab_times.sh TAG path/to/other.so [CONFIG BATCH]  (alternating, 3 rounds)
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
for r in 1 2 3; do
  echo "new $(python scripts/class_times.py ${3:-C3} ${4:-16384} 2>&1 | tail -1)" >> $OUT/ab.txt
  echo "old $(EINET_LIB_PATH=$2 python scripts/class_times.py ${3:-C3} ${4:-16384} 2>&1 | tail -1)" >> $OUT/ab.txt
done
