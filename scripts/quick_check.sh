#!/bin/bash
# Fast GPU iteration: contraction timings/trace, then the GPU suites
OUT=gpurun_out/${1:-quick}; mkdir -p $OUT
timeout 300 bash scripts/ct_diag.sh ${1:-quick}
timeout 900 python -m pytest tests -m gpu -x -q ${TESTS:-} > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt
