#!/bin/bash
# PDL on/off: bench step times at 16384, 4096, 500 (no CPU legs), then the GPU suite
OUT=gpurun_out/${1:-pdl}; mkdir -p $OUT
for pdl in 1 0 1; do
  EINET_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline --steps 50 > $OUT/bench_pdl$pdl.json 2>> $OUT/bench.err
  python -c "
import json; d=json.load(open('$OUT/bench_pdl$pdl.json'))
print('pdl=$pdl', round(d['ms_per_step'],4), [round(s['ms_per_step'],4) for s in d['secondary_batches']], round(d['e2e']['value']/1e6,2))" >> $OUT/summary.txt
done
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt
