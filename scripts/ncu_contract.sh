#!/bin/bash
# one dense-sampled ncu capture of the contraction kernels (forward layer L=4 and a child-rho pass)
OUT=gpurun_out/${1:-ncuct}; mkdir -p $OUT
EINET_LEAF_COND=0 timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on \
  -k "regex:${KREGEX:-k_contract_tc}" -s ${SKIP:-1} -c ${COUNT:-2} -o $OUT/ct python scripts/class_times.py > $OUT/ncu.log 2>&1
echo "rc=$?" >> $OUT/status.txt
