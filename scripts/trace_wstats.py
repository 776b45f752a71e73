"""Run one C3 EM step with EINET_WS_TRACE set (diagnostics for the W-statistics pipeline)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2004_06231_b200 import engine, trainer
from paper_2004_06231_b200.compiler import compile_graph
from paper_2004_06231_b200.data import config as cfg
from paper_2004_06231_b200.model import EinetModel

rg, fam, k, gen = cfg("C3")
circuit = compile_graph(rg, k)
x = torch.from_numpy(gen(16384, seed=1).astype(np.float32)).cuda()
ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=gen(2048, seed=7).astype(np.float64))
model = EinetModel(circuit, engine.Parameters.from_numpy(circuit, fam, ein, mix, phi), fam)
for _ in range(1):
    trainer.em_stochastic_step(model, x, 0.5, chunk=16384)
torch.cuda.synchronize()
