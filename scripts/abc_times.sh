#!/bin/bash
# per-class times of several library builds on one box: scripts/abc_times.sh TAG CONFIG BATCH lib1 lib2 ...
OUT=gpurun_out/$1; mkdir -p $OUT; cfg=$2; b=$3; shift 3
for r in 1 2; do for lib in "$@"; do
  echo "$(basename $lib) $(EINET_LIB_PATH=$lib python scripts/class_times.py $cfg $b 2>&1 | tail -1)" >> $OUT/abc.txt
done; done
