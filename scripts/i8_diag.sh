#!/bin/bash
OUT=gpurun_out/${1:-i8diag}; mkdir -p $OUT
EINET_I8_TRACE=1 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2004_06231_b200 as E
from paper_2004_06231_b200 import engine
from paper_2004_06231_b200.data import config
rg, fam, k, gen = config('C3')
c = E.compile_graph(rg, k)
x = torch.from_numpy(gen(${2:-16384}, seed=3).astype(np.float32)).cuda()
ein, mix, phi = engine.init_parameters_host(c, fam, seed=0, data=gen(512, seed=1))
p = engine.Parameters.from_numpy(c, fam, ein, mix, phi)
tr = E.forward(c, p, fam, x); torch.cuda.synchronize()
print('n_leaf', c.layers[0].__dict__.keys() if hasattr(c.layers[0],'__dict__') else '')
" > $OUT/trace.txt 2>&1
