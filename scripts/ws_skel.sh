#!/bin/bash
# W statistics skeleton (EINET_WS_DEBUG=3: copies + hand-offs only) vs ring shape / cluster size
OUT=gpurun_out/${1:-wsskel}; mkdir -p $OUT
for e in "EINET_WS_DEBUG=3" "EINET_WS_DEBUG=3 EINET_WS_QB=2 EINET_WS_STAGES=4" "EINET_WS_DEBUG=3 EINET_WS_QB=1 EINET_WS_STAGES=8" "EINET_WS_DEBUG=3 EINET_WS_NCL=2" "EINET_WS_DEBUG=3 EINET_WS_NCL=4" "EINET_WS_DEBUG=3 EINET_WS_NT=2" "EINET_WS_DEBUG=1" "EINET_WS_DEBUG=2" "EINET_WS_DEBUG=0"; do
  r=$(env $e timeout 120 python scripts/class_times.py C3 16384 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d.get('einsum_wstats'))")
  echo "$e wstats=$r" >> $OUT/skel.txt
done
