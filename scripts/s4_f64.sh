#!/bin/bash
# f64 host-input path: GPU suite (incl. the f64 EM tests) and the bench line.
set -u
OUT=gpurun_out/s4f; mkdir -p $OUT
nproc > $OUT/nproc.txt; lscpu | head -20 >> $OUT/nproc.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt
