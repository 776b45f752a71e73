#!/bin/bash
# W statistics: L2 prefetch distance x ring shape x tiles per segment (C3 per-class times)
OUT=gpurun_out/${1:-wspf}; mkdir -p $OUT
for cfg in "0 0 0 0" "2 0 0 0" "4 0 0 0" "4 2 4 0" "8 2 4 0" "0 0 0 2" "4 0 0 2" "4 2 6 2" "8 1 8 2"; do
  set -- $cfg
  for b in 16384 4096; do
    r=$(EINET_WS_NCL=1 EINET_WS_PREFETCH=$1 EINET_WS_QB=$2 EINET_WS_STAGES=$3 EINET_WS_NT=$4 timeout 120 python scripts/class_times.py C3 $b 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d.get('einsum_wstats'))")
    echo "pf=$1 qb=$2 st=$3 nt=$4 B=$b wstats_us=$r" >> $OUT/pf.txt
  done
done
