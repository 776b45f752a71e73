#!/bin/bash
# Final-build evidence without the profilers: smoke, GPU suite, bench line,
# reference arm, C1 / C2 small-batch lines, C4 twice per batch (its graph-replay
# time is bimodal run to run).
set -u
TAG=${1:-fin5}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/status.txt
for c in C1 C2; do timeout 300 python bench.py --config $c --batch 100 --chunk 100 --no-cpu-baseline --small-batch 0 --steps 50 > $OUT/$c.json 2>/dev/null; done
for b in 1024 4096; do
  timeout 300 python bench.py --config C4 --batch $b --chunk $b --no-cpu-baseline --small-batch 0 --steps 20 > $OUT/C4_$b.json 2>/dev/null
  timeout 300 python bench.py --config C4 --batch $b --chunk $b --no-cpu-baseline --small-batch 0 --steps 20 > $OUT/C4_${b}_b.json 2>/dev/null
done
echo done >> $OUT/status.txt
