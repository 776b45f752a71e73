#!/bin/bash
# W-statistics smem ring shapes (EINET_WS_QB blocks per unit x EINET_WS_STAGES):
# per-class times on C3 at three batches. scripts/ws_sweep.sh TAG
OUT=gpurun_out/${1:-wssweep}; mkdir -p $OUT
for cfg in "0 0" "4 2" "2 2" "2 4" "3 3" "1 4" "1 8" "2 3" "1 6"; do
  set -- $cfg
  for b in 16384 4096 500; do
    r=$(EINET_WS_QB=$1 EINET_WS_STAGES=$2 timeout 120 python scripts/class_times.py C3 $b 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d.get('einsum_wstats'))")
    echo "qb=$1 stages=$2 B=$b wstats_us=$r" >> $OUT/sweep.txt
  done
done
