#!/bin/bash
# Session-4 validation: smoke, GPU suite, bench line, per-class times at the
# secondary batches and the small-batch configs.
set -u
OUT=gpurun_out/s4; mkdir -p $OUT
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt
for b in 4096 500; do timeout 120 python scripts/class_times.py C3 $b > $OUT/class_C3_$b.txt 2>&1; done
timeout 120 python scripts/class_times.py C1 100 > $OUT/class_C1_100.txt 2>&1
timeout 120 python scripts/class_times.py C2 100 > $OUT/class_C2_100.txt 2>&1
for c in C1 C2; do timeout 300 python bench.py --config $c --batch 100 --chunk 100 --no-cpu-baseline --small-batch 0 --steps 50 > $OUT/$c.json 2>/dev/null; done
EINET_LEAF_COND=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 260 -c 60 --csv \
  --log-file $OUT/launches_500.csv python bench.py --steps 2 --warmup 3 --batch 500 --chunk 500 --no-cpu-baseline --small-batch 0 > $OUT/launches.log 2>&1
echo "launches rc=$?" >> $OUT/status.txt
