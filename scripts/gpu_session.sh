#!/bin/bash
# One gpurun call: GPU tests, bench (with CPU baseline), ncu launch list and
# one --set full capture of the top kernels. Usage: scripts/gpu_session.sh TAG [what...]
# what: tests bench launches full ref  (default: all but ref)
set -u
TAG=${1:-run}; shift || true
WHAT=${*:-tests bench launches full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
make -q -C paper_2004_06231_b200/csrc > /dev/null 2>&1 || echo "WARNING: libeinet_b200.so older than its sources" >> $OUT/status.txt
for w in $WHAT; do
case $w in
tests)
  timeout ${TEST_TIMEOUT:-400} python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt ;;
bench)
  timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt ;;
ref)
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/status.txt ;;
launches)
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 100 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/launches.log 2>&1
  echo "launches rc=$?" >> $OUT/status.txt ;;
full)
  timeout 900 ncu --set full --clock-control none --import-source on -s 10 -c ${NCU_COUNT:-8} \
    -k "regex:${NCU_KERNELS:-k_leaf_fwd_dmma|k_contract_tc|k_wstats_tc|k_leaf_stats_tc}" \
    -o $OUT/full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/full.log 2>&1
  echo "full rc=$?" >> $OUT/status.txt ;;
esac
done
