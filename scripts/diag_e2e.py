"""Where does the pipelined e2e step lose time against the device step? (diagnostic)"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_06231_b200 import engine, trainer  # noqa: E402
from paper_2004_06231_b200.compiler import compile_graph  # noqa: E402
from paper_2004_06231_b200.data import config  # noqa: E402
from paper_2004_06231_b200.model import EinetModel  # noqa: E402

rg, fam, k, gen = config("C3")
circuit = compile_graph(rg, k)
B = 16384
x64 = gen(B, seed=1)
xd = torch.from_numpy(x64.astype(np.float32)).cuda()
xu = torch.from_numpy(np.rint(x64 * 255).astype(np.uint8)).pin_memory()
ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=x64[:4096])
m = EinetModel(circuit, engine.Parameters.from_numpy(circuit, fam, ein, mix, phi), fam)
N = 50


def ev_time(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / N


def replays():
    for _ in range(N):
        trainer._graph_step(m, xd, 0.5, 1e-12, 16384, sticky=True)


eng, ws, stats, status, root = m.step_buffers(16384)
log = torch.empty((N, 2), dtype=torch.float64, device="cuda")


def replays_logged():
    for i in range(N):
        e, s, st = trainer._graph_step(m, xd, 0.5, 1e-12, 16384, sticky=True)
        log[i].copy_(s[:2])
        m.params.mark_compute_current(e)


print("graph replays only      %.3f ms/step" % ev_time(replays))
print("+ per-step log copies   %.3f ms/step" % ev_time(replays_logged))
print("em_stochastic_steps u8  %.3f ms/step" % ev_time(
    lambda: trainer.em_stochastic_steps(m, [xu] * N, 0.5, chunk=16384)))
t = time.perf_counter()
trainer.em_stochastic_steps(m, [xu] * N, 0.5, chunk=16384)
torch.cuda.synchronize()
print("  host wall             %.3f ms/step" % ((time.perf_counter() - t) * 1e3 / N))
