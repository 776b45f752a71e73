#!/bin/bash
# End-of-round evidence: smoke, GPU suite, bench line (+ reference arm), ncu
# launch list with DRAM bytes (graph conditional nodes off) and one --set full
# capture of the heavy kernels, C1/C2 small-batch lines, C4, the C5 sweep
# (3xBF16 and the single-term forward).
set -u
TAG=${1:-final}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/status.txt
for c in C1 C2; do timeout 300 python bench.py --config $c --batch 100 --chunk 100 --no-cpu-baseline --small-batch 0 --steps 50 > $OUT/$c.json 2>/dev/null; done
timeout 900 python scripts/sweep_c5.py --reps 5 --out $OUT/c5.jsonl > $OUT/c5.log 2>&1; echo "c5 rc=$?" >> $OUT/status.txt
EINET_CONTRACT_TERMS=1 timeout 600 python scripts/sweep_c5.py --ks 16,40,64 --reps 5 --out $OUT/c5_single.jsonl > $OUT/c5_single.log 2>&1
for b in 1024 4096; do timeout 300 python bench.py --config C4 --batch $b --chunk $b --no-cpu-baseline --small-batch 0 --steps 20 > $OUT/C4_$b.json 2>/dev/null; done
EINET_LEAF_COND=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 260 -c 60 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --small-batch 0 > $OUT/launches.log 2>&1
echo "launches rc=$?" >> $OUT/status.txt
EINET_LEAF_COND=0 timeout 1200 ncu --set full --clock-control none --import-source on -s 10 -c ${NCU_COUNT:-5} \
  -k "regex:${NCU_KERNELS:-k_leaf_fwd_i8|k_contract_tc|k_wstats_tc|k_leaf_stats_tc}" \
  -o $OUT/full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --small-batch 0 > $OUT/full.log 2>&1
echo "full rc=$?" >> $OUT/status.txt
