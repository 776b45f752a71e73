#!/bin/bash
# A/B of the in-tree build against build_ab/lib_base.so (bench step times at
# 16384 and the secondary batches, three alternations), then the GPU suite on
# the in-tree build.
set -u
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
for r in 1 2 3; do for lib in build_ab/lib_base.so paper_2004_06231_b200/libeinet_b200.so; do
  EINET_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 50 > $OUT/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('$OUT/b.json'))
k=d['kernels']
print('$lib'[:24], round(d['ms_per_step']*1e3,1), [round(s['ms_per_step']*1e3,1) for s in d['secondary_batches']], {c: round(k[c]['ms_per_step']*1e3,1) for c in ('leaf_stats','einsum_wstats','leaf_fwd','mixing_fwd','mixing_bwd','einsum_bwd_rt','leaf_rho','einsum_prep')})" >> $OUT/ab.txt
done; done
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt
