#!/bin/bash
# Contraction-kernel diagnostics (C3, 16384): per-class times with the
# epilogue math off (EINET_CT_DEBUG=1) / the MMAs off (=2), and the per-job
# timeline of CTA 0 (EINET_CT_TRACE) in each mode.
OUT=gpurun_out/${1:-ctdiag}; mkdir -p $OUT
python scripts/class_times.py > $OUT/base.json 2>&1
EINET_CT_DEBUG=1 python scripts/class_times.py > $OUT/noepi.json 2>&1
EINET_CT_DEBUG=2 python scripts/class_times.py > $OUT/nomma.json 2>&1
for mode in 0 1 2; do
EINET_CT_DEBUG=$mode EINET_CT_TRACE=1 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import engine
from paper_2004_06231_b200.data import config
rg, fam, k, gen = config('C3')
c = E.compile_graph(rg, k)
x = torch.from_numpy(gen(16384, seed=3).astype(np.float32)).cuda()
ein, mix, phi = engine.init_parameters_host(c, fam, seed=0, data=gen(512, seed=1))
p = engine.Parameters.from_numpy(c, fam, ein, mix, phi)
tr = E.forward(c, p, fam, x); E.backward(c, p, fam, tr); torch.cuda.synchronize()
" > $OUT/trace$mode.txt 2>&1
done
