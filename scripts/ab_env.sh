#!/bin/bash
# A/B of one environment toggle on the in-tree build: scripts/ab_env.sh TAG VAR
# (VAR=0 against unset), three alternations, then the GPU suite.
set -u
OUT=gpurun_out/$1; mkdir -p $OUT; VAR=$2
for r in 1 2 3; do for v in 0 1; do
  if [ $v = 0 ]; then export $VAR=0; else unset $VAR; fi
  timeout 300 python bench.py --no-cpu-baseline --steps 50 > $OUT/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('$OUT/b.json'))
k=d['kernels']
print('$VAR=$v', round(d['ms_per_step']*1e3,1), [round(s['ms_per_step']*1e3,1) for s in d['secondary_batches']], {c: round(k[c]['ms_per_step']*1e3,1) for c in ('leaf_stats','leaf_fwd','leaf_rho')})" >> $OUT/ab.txt
done; done
unset $VAR
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt
EINET_LEAF_COND=0 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:${KREGEX:-k_leaf_stats_tc} -c 2 --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --small-batch 0 > $OUT/ncu_on.csv 2>/dev/null
env $VAR=0 EINET_LEAF_COND=0 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:${KREGEX:-k_leaf_stats_tc} -c 2 --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --small-batch 0 > $OUT/ncu_off.csv 2>/dev/null
